"""C5 tensor-size sweep: each size class through the engine
with the gather kernel and with the copy engines, threshold below the class so
every tensor takes the D2H path. One JSON line per (class, variant)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_10707_b200 as lz  # noqa: E402
from paper_2406_10707_b200.workloads import sweep_class  # noqa: E402

total = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 30
classes = [4096, 65536, 1 << 20, 16 << 20, 256 << 20, 1 << 30]
for size in classes:
    w = sweep_class(size, max(total, 2 * size))
    built = lz.build_workload(w.write_spec(f"/tmp/sw_{size}.spec"), 0)
    cfg = lz.EngineConfig(checkpoint_root="/tmp/sw", host_buffer_bytes=int(built.bytes * 1.05) + (64 << 20),
                          large_leaf_threshold=min(4096, size), fsync_on_finalize=False, flush_discard=True,
                          hugepages=True)
    eng = lz.Engine(cfg, built.topo, built.rank)
    plan = lz.plan_checkpoint(built.topo, built.model, built.step)
    for variant in ("kernel", "copy_engine"):
        eng.set_copy_variant(force_kernel=variant == "kernel", force_copy_engine=variant == "copy_engine")
        res = []
        for s in range(3):
            h0 = time.perf_counter()
            t = eng.capture(plan, built.tree, s + 1)
            h1 = time.perf_counter()
            eng.update_barrier(t)
            dt = time.perf_counter() - h0
            eng.wait_persisted(t)
            if s:
                res.append((t.payload_bytes(), dt, eng.ticket_device_ms(t) * 1e-3, h1 - h0))
        p = res[0][0]
        print(json.dumps({"class_bytes": size, "tensors": len(w.leaves) - 1, "variant": variant, "payload": p,
                          "host_gbps": round(p * len(res) / sum(r[1] for r in res) / 1e9, 3),
                          "device_gbps": round(p * len(res) / sum(r[2] for r in res) / 1e9, 3),
                          "capture_ms": round(1e3 * sum(r[3] for r in res) / len(res), 3)}), flush=True)
    eng.close()
    del built
