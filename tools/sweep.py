"""C5 tensor-size sweep (BASELINE.json configs[4]): every
size class 4 KiB .. 1 GiB through the engine with the gather kernel and with
the copy engines (threshold below the class so every tensor takes the D2H
path). Runs on N GPUs under torchrun (one rank per GPU, all ranks sweeping
concurrently); rank 0 prints one JSON line per (class, variant) with the
per-rank and aggregate (sum of bytes / max time) GB/s.

    python tools/sweep.py [bytes_per_class]
    python -m torch.distributed.run --nproc-per-node N tools/sweep.py
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_10707_b200 as lz  # noqa: E402
from paper_2406_10707_b200.workloads import sweep_class  # noqa: E402

total = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 30
rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
dev = int(os.environ.get("LOCAL_RANK", 0))
dist = None
if world > 1:
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")  # NCCL logs off stdout
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(dev)
    sys.stdout.flush()
    saved = os.dup(1)
    os.dup2(2, 1)  # NCCL's version line goes to fd 1 at the default WARN level
    try:
        dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        dist.barrier()
    finally:
        sys.stdout.flush()
        os.dup2(saved, 1)
        os.close(saved)


def reduce(x, op):
    if dist is None:
        return x
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=op)
    return float(t.item())


# BASELINE configs[4]: "10k small tensors to few huge"
classes = [(4096, 10_000), (65536, 10_000), (1 << 20, 1024), (16 << 20, 64), (256 << 20, 4), (1 << 30, 2)]
for size, count in classes:
    w = sweep_class(size, min(total, size * count) if size < (1 << 20) else max(total, 2 * size))
    built = lz.build_workload(w.write_spec(f"/tmp/sw_{rank}_{size}.spec"), dev)
    cfg = lz.EngineConfig(checkpoint_root=f"/tmp/sw{rank}", host_buffer_bytes=int(built.bytes * 1.05) + (64 << 20),
                          large_leaf_threshold=min(4096, size), fsync_on_finalize=False, flush_discard=True,
                          hugepages=True, device=dev)
    eng = lz.Engine(cfg, built.topo, built.rank)
    plan = lz.plan_checkpoint(built.topo, built.model, built.step)
    for variant in ("kernel", "copy_engine"):
        eng.set_copy_variant(force_kernel=variant == "kernel", force_copy_engine=variant == "copy_engine")
        res = []
        for s in range(4):
            if dist is not None:
                torch.cuda.synchronize()
                dist.barrier()
            h0 = time.perf_counter()
            t = eng.capture(plan, built.tree, s + 1)
            h1 = time.perf_counter()
            eng.update_barrier(t)
            dt = time.perf_counter() - h0
            eng.wait_persisted(t)
            if s:
                res.append((t.payload_bytes(), dt, eng.ticket_device_ms(t) * 1e-3, h1 - h0))
        p = res[0][0]
        host_s = sum(r[1] for r in res)
        dev_s = sum(r[2] for r in res)
        agg_bytes = reduce(float(p * len(res)), dist.ReduceOp.SUM if dist else None)
        t_max = reduce(host_s, dist.ReduceOp.MAX if dist else None)
        t_dev_max = reduce(dev_s, dist.ReduceOp.MAX if dist else None)
        if rank == 0:
            print(json.dumps({"n_gpus": world, "class_bytes": size, "tensors": len(w.leaves) - 1, "variant": variant,
                              "payload_per_gpu": p,
                              "host_gbps_rank0": round(p * len(res) / host_s / 1e9, 3),
                              "device_gbps_rank0": round(p * len(res) / dev_s / 1e9, 3),
                              "aggregate_host_gbps": round(agg_bytes / t_max / 1e9, 3),
                              "aggregate_device_gbps": round(agg_bytes / t_dev_max / 1e9, 3),
                              "capture_ms": round(1e3 * sum(r[3] for r in res) / len(res), 3)}), flush=True)
    eng.close()
    del built
if dist is not None:
    dist.destroy_process_group()
