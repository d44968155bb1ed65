"""Host-side logic of the N>1 path on CPU with gloo, world size 2: each rank
derives its own shard plan from a dp=N topology (bench.py weak scaling), the
ranks' shard files are disjoint and together cover the whole model, every
rank's workload matches its plan exactly, and the timing reduction is a max
over ranks."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2406_10707_b200 as lz
    from paper_2406_10707_b200.workloads import llama7b_shard
    w = llama7b_shard(layers=2, vocab=1000, dp=world, rank=rank)
    topo = lz.ParallelTopology(*w.topology)
    plan = lz.plan_checkpoint(topo, lz.ModelSpec(param_count=w.param_count, layer_count=w.layer_count,
                                                 bytes_per_param_model=w.bpp_model,
                                                 bytes_per_param_optimizer=w.bpp_opt), 1)
    mine = plan.shards(rank)
    # the rank's tree (top-level children in name order) matches its shards
    tops = sorted({p.split("/")[0] for _, p, _ in w.leaves})
    sizes = [sum(s for _, p, s in w.leaves if p.split("/")[0] == t) for t in tops]
    assert sizes == [s.size_bytes for s in mine]
    files = [f"rank-{s.owner.dp}-{s.owner.pp}-{s.owner.tp}/{s.filename}" for s in mine]
    gathered = [None] * world
    dist.all_gather_object(gathered, (files, sum(sizes)))
    # weak-scaling timing: each rank's step time, reduced as the max
    t = torch.tensor([1.0 + rank], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        out.put((gathered, float(t.item()), plan.total_bytes()))
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_plans_are_disjoint_and_complete():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    gathered, tmax, total = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    all_files = [f for files, _ in gathered for f in files]
    assert len(all_files) == len(set(all_files)) == 2 * world
    assert sum(b for _, b in gathered) == total
    assert tmax == 2.0


def _commit_worker(rank, world, port, root, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2406_10707_b200.commit import distributed_commit
    manifest = os.path.join(root, "manifest.json")

    def vote(step, ok):
        files = [[f"step-{step}/rank-{rank}-0-0/layers-{rank}-{rank}.ckpt", 100 + rank, 0xA0 + rank],
                 [f"step-{step}/rank-{rank}-0-0/optimizer-{rank}.ckpt", 200 + rank, 0xB0 + rank]]
        return {"rank": rank, "step": step, "vote": "prepared" if ok else "failed",
                "detail": "" if ok else "checksum mismatch in entry 'w'", "files": files if ok else []}

    r1 = distributed_commit(None, None, None, manifest, prepare_fn=lambda: vote(3, True))
    r2 = distributed_commit(None, None, None, manifest, prepare_fn=lambda: vote(4, rank == 0))
    out.put((rank, r1, r2))
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_distributed_commit(tmp_path):
    """paper_2406_10707_b200/commit.py over gloo: votes gathered to rank 0,
    the reference coordinator's decision (consolidation.cpp:229-283), the
    manifest made durable by rank 0 before the decision is broadcast; an
    aborted step blames the failing rank and leaves the manifest untouched."""
    import json
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_commit_worker, args=(r, world, port, str(tmp_path), q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        rank, r1, r2 = q.get(timeout=240)
        res[rank] = (r1, r2)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank in range(world):
        r1, r2 = res[rank]
        assert r1.committed and r1.step == 3
        assert not r2.committed and r2.problem_ranks == [1]
        assert r2.reason == "rank 1: checksum mismatch in entry 'w'"
    m = json.load(open(tmp_path / "manifest.json"))
    assert [s["step"] for s in m["steps"]] == [3]
    paths = [f["path"] for f in m["steps"][0]["files"]]
    assert paths == sorted(paths) and len(paths) == 4
    assert {f["length"] for f in m["steps"][0]["files"]} == {100, 101, 200, 201}


def _relay_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench

    def gather(x):
        g = [None] * world
        dist.all_gather_object(g, x)
        return g

    my_rate = [57.0, 45.0][rank]
    rates = gather(my_rate)
    plan = bench.relay_plan(rates, "auto")
    armed = {"pairs": []}

    def arm(p):
        armed["pairs"] = p["pairs"]
        dist.barrier()

    def measure():
        # this rank's time under the armed plan: an owner moves (1 - x) of its
        # shard, a helper 1 + x, at the rank's own rate
        x_out = sum(x for o, _, x in armed["pairs"] if o == rank)
        x_in = sum(x for _, h, x in armed["pairs"] if h == rank)
        return gather((1 - x_out + x_in) / my_rate)

    base = gather(1 / my_rate)
    res = bench.tune_relay(plan, base, measure, arm)
    out.put((rank, res["pairs"], armed["pairs"]))
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_relay_tuning_agrees():
    """bench.py's relay planning at N=2 over gloo: every rank derives the same
    plan from the gathered rates, tunes it against gathered per-rank times, and
    arms the same final plan (the slower rank hands a share to the faster)."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_relay_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        rank, pairs, armed = q.get(timeout=240)
        res[rank] = (pairs, armed)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0] == res[1]
    pairs, armed = res[0]
    assert pairs == armed and [(o, h) for o, h, _ in pairs] == [(1, 0)]
    x = pairs[0][2]
    assert 0.05 < x < 0.2  # near the equalising share (57 - 45) / (57 + 45) = 0.118
