"""capture() is ordered after the trainer's queued writes (no host sync).

The reference serialises snapshot reads against writes under the region
mutex (/root/reference/proj/core/src/transfer_engine.cpp:10-36) and records
the captured version at submit (:77); inline leaves are cloned at capture
(engine.cpp:138-143). A capture therefore always reflects every write issued
before it. Here the writes are asynchronous kernels on the trainer's CUDA
stream, so capture(..., producer_stream) makes every snapshot read (the
inline gather, the gather kernel and the copy-engine DMAs) wait on the device
for that stream. These tests queue a ~100 ms kernel followed by rewrites of
wrapped tensors of all three size classes on a torch stream, call capture()
with NO host synchronisation, and require the files to equal the oracle's
composition of the POST-kernel state.
"""
import os
import shutil

import numpy as np
import pytest

from cases import _case

pytestmark = pytest.mark.gpu

THR = 1 << 20                 # large_leaf_threshold
INLINE = 64 << 10             # < THR: gathered into __meta__ at capture
KERNEL = (3 << 20) // 2       # THR <= size < ce_threshold (2 MiB): gather kernel
PARAMS = 8 << 20              # layers file 16 MiB, optimizer file 96 MiB (2+12 B/param)
SLEEP_CYCLES = 200_000_000    # ~100 ms at 1.9 GHz

VARIANTS = {
    "default": {},
    "kernel-only": {"force_kernel": True},
    "copy-engine-only": {"force_copy_engine": True},
    "streaming": {"stream_segment_bytes": 5_000_011, "host_buffer_bytes": 12_000_000},
}


@pytest.fixture(scope="module")
def torch_cuda(lz):
    torch = pytest.importorskip("torch")
    assert lz.device_count() > 0 and torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch


def workload():
    # layers: one inline leaf, one kernel-class leaf, the copy-engine-class rest;
    # optimizer: an inline leaf and a copy-engine-class rest
    return _case("ordering", PARAMS, 2, [
        ("layers", [("r", "small", INLINE), ("r", "mid", KERNEL), ("r", "big", None)]),
        ("optim", [("r", "m", INLINE), ("r", "v", None)]),
    ], THR)


def setup(lz, torch, w):
    """Wrapped torch tensors at zero, plus post-kernel contents already on the
    device (random bytes) and on the host for the oracle."""
    rng = np.random.default_rng(17)
    tensors, sources, post = [], [], []
    tree = lz.StateTree()
    for kind, path, size in w.leaves:
        assert kind == "r"
        t = torch.zeros(size, dtype=torch.uint8, device="cuda")
        b = rng.integers(0, 256, size, dtype=np.uint8)
        tensors.append(t)
        sources.append(torch.from_numpy(b).cuda())
        post.append(b)
        tree.set_region(path, lz.DeviceRegion.wrap(t))
    torch.cuda.synchronize()
    return tree, tensors, sources, post


def queue_rewrite(torch, stream, tensors, sources):
    """A ~100 ms kernel, then every tensor rewritten, all on `stream`; the host
    returns immediately."""
    with torch.cuda.stream(stream):
        torch.cuda._sleep(SLEEP_CYCLES)
        for t, s in zip(tensors, sources):
            t.copy_(s)


def files_of(t, root):
    return {os.path.relpath(f, root): np.fromfile(f, dtype=np.uint8) for f in t.shard_files()}


@pytest.mark.parametrize("variant", list(VARIANTS))
@pytest.mark.parametrize("which", ["current", "side"])
def test_capture_reads_post_kernel_state_without_host_sync(lz, torch_cuda, oracle, tmp_path, variant, which):
    torch = torch_cuda
    w, thr = workload()
    tree, tensors, sources, post = setup(lz, torch, w)
    knobs = dict(VARIANTS[variant])
    pool = knobs.pop("host_buffer_bytes", 256 << 20)
    root = tmp_path / "ckpt"
    eng = lz.Engine(lz.EngineConfig(checkpoint_root=str(root), host_buffer_bytes=pool, large_leaf_threshold=thr,
                                    fsync_on_finalize=False, **knobs),
                    lz.ParallelTopology(1, 1, 1, 1, 1), lz.RankCoord())
    plan = lz.plan_checkpoint(lz.ParallelTopology(1, 1, 1, 1, 1), lz.ModelSpec(param_count=w.param_count, layer_count=w.layer_count), 1)
    stream = torch.cuda.current_stream() if which == "current" else torch.cuda.Stream()
    queue_rewrite(torch, stream, tensors, sources)
    assert not stream.query(), "the rewrite must still be running when capture() is called"
    if which == "current":
        t = eng.capture(plan, tree, 1)  # default producer: torch's current stream
    else:
        t = eng.capture(plan, tree, 1, producer_stream=stream)
    eng.update_barrier(t)
    eng.wait_persisted(t)
    assert t.status() == "persisted" and not t.torn()
    expect = oracle.compose_files(w, thr, data=post)
    got = files_of(t, root)
    assert set(got) == set(expect)
    for rel in expect:
        assert np.array_equal(got[rel], expect[rel]), (variant, rel)
    eng.close()
    shutil.rmtree(root, ignore_errors=True)


def test_unordered_capture_reads_stale_bytes(lz, torch_cuda, oracle, tmp_path):
    """Control: the reference-signature capture (producer_stream=None) does not
    wait for the trainer's stream, so the same race is visible — this is the
    bug the ordered capture removes, not a property anyone should rely on."""
    torch = torch_cuda
    w, thr = workload()
    tree, tensors, sources, post = setup(lz, torch, w)
    root = tmp_path / "ckpt"
    eng = lz.Engine(lz.EngineConfig(checkpoint_root=str(root), host_buffer_bytes=256 << 20,
                                    large_leaf_threshold=thr, fsync_on_finalize=False),
                    lz.ParallelTopology(1, 1, 1, 1, 1), lz.RankCoord())
    plan = lz.plan_checkpoint(lz.ParallelTopology(1, 1, 1, 1, 1), lz.ModelSpec(param_count=w.param_count, layer_count=w.layer_count), 1)
    s = torch.cuda.Stream()
    queue_rewrite(torch, s, tensors, sources)
    t = eng.capture(plan, tree, 1, producer_stream=None)
    eng.update_barrier(t)
    eng.wait_persisted(t)
    want = oracle.compose_files(w, thr, data=post)
    got = files_of(t, root)
    # the inline leaves were cloned synchronously before the rewrite ran
    assert any(not np.array_equal(got[rel], want[rel]) for rel in want)
    s.synchronize()
    eng.close()


def test_fence_then_optimizer_step_without_host_sync(lz, torch_cuda, oracle, tmp_path):
    """The whole no-sync loop: rewrite (step k) -> capture -> device fence ->
    rewrite again (step k+1) on the same stream, for three steps; each
    checkpoint holds exactly its own step's state."""
    torch = torch_cuda
    w, thr = workload()
    tree, tensors, sources, post = setup(lz, torch, w)
    root = tmp_path / "ckpt"
    eng = lz.Engine(lz.EngineConfig(checkpoint_root=str(root), host_buffer_bytes=512 << 20,
                                    large_leaf_threshold=thr, fsync_on_finalize=False),
                    lz.ParallelTopology(1, 1, 1, 1, 1), lz.RankCoord())
    topo = lz.ParallelTopology(1, 1, 1, 1, 1)
    model = lz.ModelSpec(param_count=w.param_count, layer_count=w.layer_count)
    s = torch.cuda.Stream()
    tickets, states = [], []
    for step in range(1, 4):
        with torch.cuda.stream(s):
            torch.cuda._sleep(SLEEP_CYCLES // 4)
            for t_, src in zip(tensors, sources):
                t_.add_(src)  # "optimizer step": state_k = k * src (mod 256)
        states.append([(np.uint16(step) * p).astype(np.uint8) for p in post])
        k = eng.capture(lz.plan_checkpoint(topo, model, step), tree, step, producer_stream=s)
        eng.update_barrier_on_stream(k, s.cuda_stream)  # the next step waits for the snapshot
        tickets.append(k)
    for step, (k, state) in enumerate(zip(tickets, states), start=1):
        eng.wait_persisted(k)
        assert not k.torn()
        w.step = step
        expect = oracle.compose_files(w, thr, data=state)
        got = files_of(k, root)
        for rel in expect:
            assert np.array_equal(got[rel], expect[rel]), (step, rel)
    s.synchronize()
    eng.close()


def test_checkpoint_engine_save_right_after_step(lz, torch_cuda, tmp_path):
    """DeepSpeed-style save() right after an un-synchronised optimizer step:
    the file holds the updated parameters and Adam moments."""
    torch = torch_cuda
    from paper_2406_10707_b200.checkpoint_engine import DataStatesCheckpointEngine
    torch.manual_seed(0)
    model = torch.nn.Sequential(torch.nn.Linear(1024, 4096), torch.nn.GELU(), torch.nn.Linear(4096, 1024)).cuda()
    opt = torch.optim.Adam(model.parameters(), lr=1e-3)
    x = torch.randn(256, 1024, device="cuda")
    ce = DataStatesCheckpointEngine(host_cache_bytes=256 << 20, large_leaf_threshold=THR,
                                    config_params={"fsync": False})
    path = str(tmp_path / "ck.lzckpt")
    for _ in range(2):
        opt.zero_grad(set_to_none=True)
        model(x).square().mean().backward()
        torch.cuda._sleep(SLEEP_CYCLES // 2)  # keep the device busy behind the host
        opt.step()
    state = {"model": model.state_dict(), "optim": opt.state_dict()}
    ce.save(state, path)  # no synchronize() before it
    ce.wait()
    ce.commit()
    want = {k: v.detach().cpu().clone() for k, v in model.state_dict().items()}
    back = ce.load(path)
    for k, v in want.items():
        assert torch.equal(back["model"][k].cpu(), v), k
    for i, st in opt.state_dict()["state"].items():
        for name in ("exp_avg", "exp_avg_sq"):
            assert torch.equal(back["optim"]["state"][i][name].cpu(), st[name].cpu()), (i, name)
