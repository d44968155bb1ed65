"""Uplink relay between two ranks (two processes, two GPUs): the owner (this
process, cuda:0) delegates a suffix of each shard file's large leaves to a
helper process on cuda:1, which reads them from the owner's HBM through CUDA
IPC (NVLink) with its copy engines (or its gather kernel), stores them through
its own PCIe link and writes them into the owner's files (relay.hpp). Both
helper routes run every test. The files must be
byte-identical to the oracle's composition, with the header still written
last by the owner; the capture stays ordered after the owner's trainer stream
across the process boundary (interprocess event). Needs two GPUs; skipped
otherwise (the driver's single-GPU run), exercised with `gpurun --gpus 2`."""
import os
import subprocess
import sys
import time

import numpy as np
import pytest

from cases import _case

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HELPER = r"""
import os, sys, time
sys.path.insert(0, os.environ["LZK_ROOT"])
import paper_2406_10707_b200 as lz
cfg = lz.EngineConfig(checkpoint_root=os.environ["LZK_TMP"], host_buffer_bytes=64 << 20, device=1,
                      relay_serve_socket=os.environ["LZK_SOCK"], relay_staging_bytes=64 << 20,
                      relay_kernel_route=os.environ.get("LZK_ROUTE") == "kernel")
eng = lz.Engine(cfg, lz.ParallelTopology(1, 1, 1, 1, 1), lz.RankCoord())
open(os.environ["LZK_SOCK"] + ".ready", "w").close()
while not os.path.exists(os.environ["LZK_SOCK"] + ".stop"):
    time.sleep(0.05)
print("served", eng.relay_stats(), flush=True)
eng.close()
"""


def workload():
    # layers 16 MiB, optimizer 96 MiB (2+12 B/param); the last large leaf of
    # each file fits a 0.6 share of its payload and moves to the helper
    return _case("relay", 8 << 20, 2, [
        ("layers", [("r", "small", 64 << 10), ("r", "a", 3 << 20), ("r", "b", 5 << 20), ("r", "c", None)]),
        ("optim", [("r", "m", 64 << 10), ("r", "v1", 20 << 20), ("r", "v2", 30 << 20), ("r", "v3", None)]),
    ], 1 << 20)


@pytest.fixture(params=["ce", "kernel"])
def helper(tmp_path, request):
    """A helper process on cuda:1 serving the relay through its copy engines
    (D2D pull into HBM staging, then DMA; the default) or its gather kernel."""
    torch = pytest.importorskip("torch")
    if torch.cuda.device_count() < 2:
        pytest.skip("the relay needs two GPUs (run with gpurun --gpus 2)")
    sock = str(tmp_path / "relay.sock")
    env = dict(os.environ, LZK_ROOT=ROOT, LZK_TMP=str(tmp_path), LZK_SOCK=sock, LZK_ROUTE=request.param)
    p = subprocess.Popen([sys.executable, "-c", HELPER], env=env, stdout=subprocess.PIPE, stderr=subprocess.STDOUT,
                         text=True)
    t0 = time.time()
    while not os.path.exists(sock + ".ready"):
        assert p.poll() is None, p.stdout.read()
        assert time.time() - t0 < 120, "helper did not start"
        time.sleep(0.05)
    yield sock
    open(sock + ".stop", "w").close()
    out, _ = p.communicate(timeout=120)
    assert p.returncode == 0, out
    print(out)


@pytest.mark.parametrize("fsync", [False, True])
def test_relayed_files_match_the_oracle(lz, oracle, tmp_path, helper, fsync):
    torch = pytest.importorskip("torch")
    w, thr = workload()
    rng = np.random.default_rng(23)
    tree = lz.StateTree()
    tensors, sources, post = [], [], []
    for _, path, size in w.leaves:
        t = torch.zeros(size, dtype=torch.uint8, device="cuda:0")
        b = rng.integers(0, 256, size, dtype=np.uint8)
        tensors.append(t)
        sources.append(torch.from_numpy(b).to("cuda:0"))
        post.append(b)
        tree.set_region(path, lz.DeviceRegion.wrap(t))
    torch.cuda.synchronize()
    root = tmp_path / "ckpt"
    eng = lz.Engine(lz.EngineConfig(checkpoint_root=str(root), host_buffer_bytes=256 << 20, device=0,
                                    large_leaf_threshold=thr, fsync_on_finalize=fsync,
                                    relay_peer_socket=helper, relay_share=0.6, relay_min_entry=1 << 20),
                    lz.ParallelTopology(1, 1, 1, 1, 1), lz.RankCoord())
    plan = lz.plan_checkpoint(lz.ParallelTopology(1, 1, 1, 1, 1),
                              lz.ModelSpec(param_count=w.param_count, layer_count=w.layer_count), 1)
    # the rewrite is still running when capture() is called: the helper's
    # reads must wait for it (interprocess producer event)
    stream = torch.cuda.current_stream(0)
    with torch.cuda.stream(stream):
        torch.cuda._sleep(100_000_000)
        for t, s in zip(tensors, sources):
            t.copy_(s)
    t = eng.capture(plan, tree, 1)
    eng.update_barrier(t)
    eng.wait_persisted(t)
    assert t.status() == "persisted" and not t.torn()
    stats = eng.relay_stats()
    delegated = [s for (_, p, s) in w.leaves if p in ("layers/c", "optim/v3")]
    assert stats["delegated_bytes"] == sum(delegated), stats
    expect = oracle.compose_files(w, thr, data=post)
    got = {os.path.relpath(f, root): np.fromfile(f, dtype=np.uint8) for f in t.shard_files()}
    assert set(got) == set(expect)
    for rel in expect:
        assert np.array_equal(got[rel], expect[rel]), rel
    # restore validates every entry checksum, including the helper's
    m = lz.ManifestStore(str(tmp_path / "manifest.json"))
    m.commit_step(1, lz.committed_record(t, str(root)))
    back = eng.restore(m, 1)
    assert back.region_at("optim/v3").clone_bytes() == post[-1].tobytes()
    eng.close()


def test_relay_discard_tier_completes(lz, tmp_path, helper):
    """Host-memory tier (the bench's timed steps): the helper only moves the
    bytes through its link; the ticket completes and the counters add up."""
    torch = pytest.importorskip("torch")
    w, thr = workload()
    tree = lz.StateTree()
    keep = []
    for _, path, size in w.leaves:
        t = torch.full((size,), 7, dtype=torch.uint8, device="cuda:0")
        keep.append(t)
        tree.set_region(path, lz.DeviceRegion.wrap(t))
    eng = lz.Engine(lz.EngineConfig(checkpoint_root=str(tmp_path / "d"), host_buffer_bytes=256 << 20, device=0,
                                    large_leaf_threshold=thr, flush_discard=True, fsync_on_finalize=False,
                                    relay_peer_socket=helper, relay_share=0.6, relay_min_entry=1 << 20),
                    lz.ParallelTopology(1, 1, 1, 1, 1), lz.RankCoord())
    plan = lz.plan_checkpoint(lz.ParallelTopology(1, 1, 1, 1, 1),
                              lz.ModelSpec(param_count=w.param_count, layer_count=w.layer_count), 1)
    for step in range(1, 4):
        t = eng.capture(plan, tree, step)
        eng.update_barrier(t)
        eng.wait_persisted(t)
        assert not t.torn()
    assert eng.relay_stats()["delegated_bytes"] > 0
    eng.close()


def test_relay_tear_is_detected(lz, tmp_path, helper):
    """A delegated leaf mutated (declared) before the helper has read it tears
    the ticket, as a local copy would (reference transfer_engine.cpp:146-154):
    the helper's read waits behind a 100 ms kernel on the producer stream."""
    torch = pytest.importorskip("torch")
    w, thr = workload()
    tree = lz.StateTree()
    regions, keep = {}, []
    for _, path, size in w.leaves:
        t = torch.zeros(size, dtype=torch.uint8, device="cuda:0")
        keep.append(t)
        regions[path] = lz.DeviceRegion.wrap(t)
        tree.set_region(path, regions[path])
    torch.cuda.synchronize()
    eng = lz.Engine(lz.EngineConfig(checkpoint_root=str(tmp_path / "t"), host_buffer_bytes=256 << 20, device=0,
                                    large_leaf_threshold=thr, fsync_on_finalize=False,
                                    relay_peer_socket=helper, relay_share=0.6, relay_min_entry=1 << 20),
                    lz.ParallelTopology(1, 1, 1, 1, 1), lz.RankCoord())
    plan = lz.plan_checkpoint(lz.ParallelTopology(1, 1, 1, 1, 1),
                              lz.ModelSpec(param_count=w.param_count, layer_count=w.layer_count), 1)
    torch.cuda._sleep(200_000_000)  # the helper's read waits behind this
    t = eng.capture(plan, tree, 1)
    regions["optim/v3"].bump_version()  # a delegated leaf changes before it was read
    with pytest.raises(lz.TornSnapshot):
        eng.update_barrier(t)
    assert t.torn()
    eng.drain()
    # the file holding the torn leaf never gets a header (files of the ticket
    # that finished before the tear was seen may; the failed ticket and the
    # 2PC keep them out of any committed step, as in the reference)
    torn_file = [f for f in t.shard_files() if os.path.basename(f).startswith("optimizer")]
    assert torn_file
    with pytest.raises(lz.Error):
        lz.read_header(torn_file[0])
    eng.close()


def test_lost_helper_fails_loudly(lz, tmp_path):
    """The helper process dies: the owner's next capture raises instead of
    hanging, and closing the engine returns."""
    torch = pytest.importorskip("torch")
    if torch.cuda.device_count() < 2:
        pytest.skip("the relay needs two GPUs (run with gpurun --gpus 2)")
    sock = str(tmp_path / "relay.sock")
    env = dict(os.environ, LZK_ROOT=ROOT, LZK_TMP=str(tmp_path), LZK_SOCK=sock)
    p = subprocess.Popen([sys.executable, "-c", HELPER], env=env, stdout=subprocess.DEVNULL,
                         stderr=subprocess.DEVNULL)
    t0 = time.time()
    while not os.path.exists(sock + ".ready"):
        assert p.poll() is None and time.time() - t0 < 120
        time.sleep(0.05)
    w, thr = workload()
    tree = lz.StateTree()
    keep = []
    for _, path, size in w.leaves:
        t = torch.zeros(size, dtype=torch.uint8, device="cuda:0")
        keep.append(t)
        tree.set_region(path, lz.DeviceRegion.wrap(t))
    eng = lz.Engine(lz.EngineConfig(checkpoint_root=str(tmp_path / "l"), host_buffer_bytes=256 << 20, device=0,
                                    large_leaf_threshold=thr, fsync_on_finalize=False,
                                    relay_peer_socket=sock, relay_share=0.6, relay_min_entry=1 << 20),
                    lz.ParallelTopology(1, 1, 1, 1, 1), lz.RankCoord())
    p.kill()
    p.wait(timeout=60)
    time.sleep(0.5)  # the owner's reader sees the closed connection
    plan = lz.plan_checkpoint(lz.ParallelTopology(1, 1, 1, 1, 1),
                              lz.ModelSpec(param_count=w.param_count, layer_count=w.layer_count), 1)
    with pytest.raises(lz.Error):
        t = eng.capture(plan, tree, 1)
        eng.update_barrier(t)
        eng.wait_persisted(t)
    eng.close()
