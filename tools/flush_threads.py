"""Durable flush throughput vs flush threads on the e2e slice (C2, 2 layers,
7.5 GB, fsync on local disk).  python tools/flush_threads.py 4 8 16"""
import os
import shutil
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_10707_b200 as lz  # noqa: E402
from paper_2406_10707_b200.workloads import llama7b_shard  # noqa: E402

w = llama7b_shard(layers=2, vocab=8000, name="ft")
built = lz.build_workload(w.write_spec("/tmp/ft.spec"), 0)
plan = lz.plan_checkpoint(built.topo, built.model, built.step)
for th in [int(x) for x in sys.argv[1:]] or [8]:
    root = f"/tmp/ft_{th}"
    cfg = lz.EngineConfig(checkpoint_root=root, host_buffer_bytes=int(built.bytes * 1.01) + (64 << 20),
                          fsync_on_finalize=True, flush_threads=th)
    eng = lz.Engine(cfg, built.topo, built.rank)
    ts = []
    for s in range(3):
        h0 = time.perf_counter()
        t = eng.capture(plan, built.tree, 10 + s)
        eng.update_barrier(t)
        eng.wait_persisted(t)
        if s:
            ts.append(time.perf_counter() - h0)
        shutil.rmtree(os.path.join(root, f"step-{10 + s}"), ignore_errors=True)
    eng.close()
    shutil.rmtree(root, ignore_errors=True)
    print(f"flush_threads={th}: {built.bytes * len(ts) / sum(ts) / 1e9:.3f} GB/s durable", flush=True)
