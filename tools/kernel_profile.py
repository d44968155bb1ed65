"""Drives lzk_gather_kernel on a C5 size class through the
public engine API, for ncu: `python tools/kernel_profile.py [tensor_bytes] [total_bytes] [steps]`.
Prints the device GB/s of each step (CUDA events on the snapshot stream)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_10707_b200 as lz  # noqa: E402
from paper_2406_10707_b200.workloads import sweep_class  # noqa: E402

size = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
total = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 30
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
w = sweep_class(size, total)
built = lz.build_workload(w.write_spec(f"/tmp/kp_{size}.spec"), 0)
cfg = lz.EngineConfig(checkpoint_root="/tmp/kp", host_buffer_bytes=int(built.bytes * 1.05) + (64 << 20),
                      large_leaf_threshold=min(4096, size), fsync_on_finalize=False, flush_discard=True,
                      force_kernel=True, hugepages=True)
eng = lz.Engine(cfg, built.topo, built.rank)
plan = lz.plan_checkpoint(built.topo, built.model, built.step)
for s in range(steps):
    h0 = time.perf_counter()
    t = eng.capture(plan, built.tree, s + 1)
    eng.update_barrier(t)
    dt = time.perf_counter() - h0
    eng.wait_persisted(t)
    print(f"class {size} B x {len(w.leaves) - 1}: {t.payload_bytes() / 1e9:.2f} GB, host {t.payload_bytes() / dt / 1e9:.2f} GB/s, "
          f"device {t.payload_bytes() / (eng.ticket_device_ms(t) * 1e-3) / 1e9:.2f} GB/s, "
          f"stats {eng.snapshot_stats()}", flush=True)
