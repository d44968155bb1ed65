"""Capture-phase timing at C2 (LZCKPT_TRACE=1 prints the phases): 1164
tensors, 107.8 GB, host-memory flush tier.  python tools/cap_c2.py [layers]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_10707_b200 as lz  # noqa: E402
from paper_2406_10707_b200.workloads import llama7b_shard  # noqa: E402

layers = int(sys.argv[1]) if len(sys.argv) > 1 else 32
w = llama7b_shard(layers=layers)
built = lz.build_workload(w.write_spec("/tmp/cap_c2.spec"), 0)
cfg = lz.EngineConfig(checkpoint_root="/tmp/cap_c2", host_buffer_bytes=int(built.bytes * 1.01) + (256 << 20),
                      large_leaf_threshold=1 << 20, fsync_on_finalize=False, flush_discard=True, hugepages=True)
eng = lz.Engine(cfg, built.topo, built.rank)
plan = lz.plan_checkpoint(built.topo, built.model, built.step)
for s in range(4):
    h0 = time.perf_counter()
    t = eng.capture(plan, built.tree, s + 1)
    h1 = time.perf_counter()
    eng.update_barrier(t)
    eng.wait_persisted(t)
    print(f"capture {1e3 * (h1 - h0):.3f} ms (python call)", flush=True)
eng.close()
