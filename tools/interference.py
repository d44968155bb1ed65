"""Where the per-iteration slowdown under checkpointing comes from.
Times the bench's synthetic fwd/bwd (bf16 8192^3 GEMMs on a compute stream)
  A: alone,
  B: with a raw copy-engine D2H of the same bytes on a side stream (torch
     non_blocking copies into pinned memory; no engine, no host threads),
  C: with an Engine capture of the C2 shard (the bench's configuration),
  D: the same with every byte forced through lzk_gather_kernel (2, 4 and 8
     CTAs): the SM time the kernel variant takes from the trainer, by grid.
Prints one JSON line; B - A is hardware interference, C - B the engine's own.
    python tools/interference.py [layers]"""
import json
import os
import statistics
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_10707_b200 as lz  # noqa: E402
from paper_2406_10707_b200.workloads import llama7b_shard  # noqa: E402

layers = int(sys.argv[1]) if len(sys.argv) > 1 else 32
w = llama7b_shard(layers=layers)
built = lz.build_workload(w.write_spec("/tmp/intf.spec"), 0)
payload = built.bytes
cfg = lz.EngineConfig(checkpoint_root="/tmp/intf", host_buffer_bytes=int(payload * 1.01) + (256 << 20),
                      large_leaf_threshold=1 << 20, fsync_on_finalize=False, flush_discard=True, hugepages=True)
eng = lz.Engine(cfg, built.topo, built.rank)
plan = lz.plan_checkpoint(built.topo, built.model, built.step)

n = 8192
a = torch.randn(n, n, dtype=torch.bfloat16, device="cuda")
b = torch.randn(n, n, dtype=torch.bfloat16, device="cuda")
c = torch.empty(n, n, dtype=torch.bfloat16, device="cuda")
comp = torch.cuda.Stream()
side = torch.cuda.Stream()
for _ in range(20):
    torch.matmul(a, b, out=c)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(50):
    torch.matmul(a, b, out=c)
e1.record()
e1.synchronize()
per_mm = e0.elapsed_time(e1) / 50
n_mm = int(1.1 * payload / 57e9 * 1e3 / per_mm)

# raw DMA source/target: a 4 GiB device tensor copied repeatedly into pinned host memory
src = torch.empty(4 << 30, dtype=torch.uint8, device="cuda")
dst = torch.empty(4 << 30, dtype=torch.uint8, pin_memory=True)


def gemms():
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record(comp)
    with torch.cuda.stream(comp):
        for _ in range(n_mm):
            torch.matmul(a, b, out=c)
    s1.record(comp)
    return s0, s1


def run(mode):
    torch.cuda.synchronize()
    h0 = time.perf_counter()
    t = None
    if mode.startswith("engine"):
        kernel = mode.startswith("engine_kernel")
        ctas = int(mode.rsplit("_", 1)[1]) if kernel else 8
        eng.set_copy_variant(force_kernel=kernel, force_copy_engine=False, kernel_ctas=ctas)
        t = eng.capture(plan, built.tree, int(time.time() * 1000) % 1000000 + 1)
    elif mode == "raw_dma":
        with torch.cuda.stream(side):
            left = payload
            while left > 0:
                k = min(left, 4 << 30)
                dst[:k].copy_(src[:k], non_blocking=True)
                left -= k
    s0, s1 = gemms()
    if t is not None:
        eng.update_barrier_on_stream(t, comp.cuda_stream)
    s1.synchronize()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - h0) * 1e3
    if t is not None:
        eng.wait_persisted(t)
    return s0.elapsed_time(s1), wall


res = {}
for mode in ("alone", "raw_dma", "engine", "engine_kernel_2", "engine_kernel_4", "engine_kernel_8") * 3:
    g, wall = run(mode)
    res.setdefault(mode, []).append((g, wall))
out = {"n_mm": n_mm, "per_mm_ms": round(per_mm, 4), "payload": payload}
for k, v in res.items():
    out[k] = {"gemm_ms": round(statistics.median(x[0] for x in v), 2),
              "wall_ms": round(statistics.median(x[1] for x in v), 2)}
out["hw_interference_ms"] = round(out["raw_dma"]["gemm_ms"] - out["alone"]["gemm_ms"], 2)
out["engine_extra_ms"] = round(out["engine"]["gemm_ms"] - out["raw_dma"]["gemm_ms"], 2)
for c in (2, 4, 8):
    out[f"kernel_variant_extra_ms_{c}ctas"] = round(out[f"engine_kernel_{c}"]["gemm_ms"] - out["alone"]["gemm_ms"], 2)
print(json.dumps(out))
eng.close()
