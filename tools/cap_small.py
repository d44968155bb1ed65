import os, sys, time
sys.path.insert(0, '/root/repo')
import paper_2406_10707_b200 as lz
from paper_2406_10707_b200.workloads import sweep_class
w = sweep_class(4096, 40 << 20)
built = lz.build_workload(w.write_spec('/tmp/c4k.spec'), 0)
cfg = lz.EngineConfig(checkpoint_root='/tmp/c4k', host_buffer_bytes=int(built.bytes * 1.05) + (64 << 20),
                      large_leaf_threshold=4096, fsync_on_finalize=False, flush_discard=True, hugepages=True)
eng = lz.Engine(cfg, built.topo, built.rank)
plan = lz.plan_checkpoint(built.topo, built.model, built.step)
eng.set_copy_variant(force_kernel=True, force_copy_engine=False)
for s in range(4):
    h0 = time.perf_counter(); t = eng.capture(plan, built.tree, s + 1); h1 = time.perf_counter()
    eng.update_barrier(t); h2 = time.perf_counter(); eng.wait_persisted(t); h3 = time.perf_counter()
    print(f"capture {1e3*(h1-h0):.2f} ms barrier {1e3*(h2-h1):.2f} ms persisted {1e3*(h3-h2):.2f} ms dev {eng.ticket_device_ms(t):.2f} ms", flush=True)
eng.close()
