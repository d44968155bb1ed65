"""Which part of the Python bench process slows the D2H? Runs the engine
snapshot on C2 after progressively more of bench.py's setup."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
stage = sys.argv[1]
if stage != "none":
    import torch
    torch.cuda.set_device(0)
import paper_2406_10707_b200 as lz
from paper_2406_10707_b200.workloads import llama7b_shard
w = llama7b_shard(layers=int(sys.argv[2]) if len(sys.argv) > 2 else 32)
spec = w.write_spec("/tmp/pyb.spec")
built = lz.build_workload(spec, 0)
if stage in ("probe", "probe_free"):
    src = torch.empty(4 << 30, dtype=torch.uint8, device="cuda")
    dst = torch.empty(4 << 30, dtype=torch.uint8, pin_memory=True)
    for _ in range(3):
        dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    del src, dst
    torch.cuda.empty_cache()
    if stage == "probe_free":
        torch._C._host_emptyCache() if hasattr(torch._C, "_host_emptyCache") else None
cfg = lz.EngineConfig(checkpoint_root="/tmp/pyb", host_buffer_bytes=int(built.bytes * 1.01) + (256 << 20),
                      fsync_on_finalize=False, flush_discard=True, hugepages=True, device=0)
eng = lz.Engine(cfg, built.topo, built.rank)
plan = lz.plan_checkpoint(built.topo, built.model, built.step)
for r in range(4):
    h0 = time.perf_counter()
    t = eng.capture(plan, built.tree, 10 + r)
    eng.update_barrier(t)
    dt = time.perf_counter() - h0
    eng.wait_persisted(t)
    print(f"stage={stage} step {r}: host {t.payload_bytes()/dt/1e9:.2f} GB/s device {t.payload_bytes()/(eng.ticket_device_ms(t)*1e-3)/1e9:.2f} GB/s", flush=True)
