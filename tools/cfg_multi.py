"""BASELINE configs[0] (C1) timing and configs[2] (C3) under torchrun.
  C1: GPT-2-small shard (1.742 GB, mt19937_64(125)) snapshot GB/s, N=1;
  C3: every rank snapshots its own ~26 GB shard of a 13B dp=8 plan
      concurrently (rank r = dp rank r); per-GPU and aggregate GB/s
      (bytes of all ranks / slowest rank's time), host-memory flush tier.
One JSON line per config on rank 0.
    python -m torch.distributed.run --nproc-per-node N tools/cfg_multi.py"""
import json
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
dev = int(os.environ.get("LOCAL_RANK", 0))
import torch  # noqa: E402
torch.cuda.set_device(dev)
dist = None
if world > 1:
    import torch.distributed as dist
    sys.stdout.flush()
    saved = os.dup(1)
    os.dup2(2, 1)
    try:
        dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        dist.barrier()
    finally:
        sys.stdout.flush()
        os.dup2(saved, 1)
        os.close(saved)
import bench  # noqa: E402
import paper_2406_10707_b200 as lz  # noqa: E402
from paper_2406_10707_b200.workloads import gpt2_small, llama13b_shard  # noqa: E402


def barrier():
    torch.cuda.synchronize()
    if dist:
        dist.barrier()


def reduce(x, op):
    if not dist:
        return x
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=op)
    return float(t.item())


def snap(w, tmp, steps=4):
    built = lz.build_workload(w.write_spec(os.path.join(tmp, "w.spec")), dev)
    cfg = lz.EngineConfig(checkpoint_root=os.path.join(tmp, "ck"), host_buffer_bytes=int(built.bytes * 1.02) + (64 << 20),
                          large_leaf_threshold=1 << 20, fsync_on_finalize=False, flush_discard=True, hugepages=True,
                          device=dev)
    eng = lz.Engine(cfg, built.topo, built.rank)
    plan = lz.plan_checkpoint(built.topo, built.model, built.step)
    ts = []
    for s in range(steps):
        barrier()
        h0 = time.perf_counter()
        t = eng.capture(plan, built.tree, s + 1)
        eng.update_barrier(t)
        dt = time.perf_counter() - h0
        eng.wait_persisted(t)
        if s:
            ts.append(dt)
    eng.close()
    return built.bytes, ts


tmp = tempfile.mkdtemp(prefix=f"lzk_cfg_r{rank}_", dir=bench.ROOT)
if world == 1:
    nbytes, ts = snap(gpt2_small(), tmp)
    print(json.dumps({"config": "c1-gpt2-small (configs[0])", "payload_bytes": nbytes,
                      "gbps": round(nbytes * len(ts) / sum(ts) / 1e9, 3)}), flush=True)
nbytes, ts = snap(llama13b_shard(rank=rank), tmp)
t_max = reduce(sum(ts), dist.ReduceOp.MAX if dist else None)
agg = reduce(float(nbytes * len(ts)), dist.ReduceOp.SUM if dist else None)
if rank == 0:
    print(json.dumps({"config": f"c3-llama13b dp=8 plan, ranks 0..{world - 1} concurrently (configs[2])",
                      "n_gpus": world, "payload_bytes_per_gpu": nbytes, "per_gpu_gbps_rank0": round(nbytes * len(ts) / sum(ts) / 1e9, 3),
                      "aggregate_gbps": round(agg / t_max / 1e9, 3)}), flush=True)
import shutil  # noqa: E402
shutil.rmtree(tmp, ignore_errors=True)
if dist:
    dist.destroy_process_group()
