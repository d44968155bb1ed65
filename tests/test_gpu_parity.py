"""GPU parity: the B200 engine's shard files against the reference's own
output (tests/golden/ref_fixtures.json, produced by the reference engine) and
byte-for-byte against the oracle's composition of the same workload; the
gather/scatter kernels against numpy on random byte-granular layouts; torn
detection, the device-side lazy fence, restore and backpressure.

Everything calls through the C ABI (liblzckpt_b200.so / liblzk_cuda.so)."""
import ctypes as C
import os
import shutil
import threading
import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
C1_GOLDEN = {"step-1/rank-0-0-0/layers-0-11.ckpt": (248887594, 0x18D06AB61AFAE34A),
             "step-1/rank-0-0-0/optimizer-0.ckpt": (1493305660, 0xC1F7BF0708955268)}

# engine knob sets that must all give identical files
VARIANTS = {
    "default": {},
    "kernel-only": {"force_kernel": True},
    "copy-engine-only": {"force_copy_engine": True},
    "tiny-groups": {"group_bytes": 4096, "chunk_quantum": 1500, "kernel_ctas": 3},
    # pool far smaller than the files: every file streams through odd-sized
    # segments with backpressure (C4 mode), bytes must not change
    "streaming": {"stream_segment_bytes": 1_000_003, "host_buffer_bytes": 3_000_009, "chunk_quantum": 262_147},
    # durable files: O_DIRECT interior + buffered edge blocks + header last +
    # fsync (FlushConfig::direct_io)
    "durable": {"fsync_on_finalize": True},
    "durable-streaming": {"fsync_on_finalize": True, "stream_segment_bytes": 1_000_003,
                          "host_buffer_bytes": 3_000_009, "chunk_quantum": 262_147},
    # one writer at a time, odd small pieces (FlushConfig::max_writers / write_piece)
    "durable-one-writer": {"fsync_on_finalize": True, "flush_max_writers": 1, "flush_write_piece": 1_048_576 + 4096},
}


@pytest.fixture(scope="module")
def gpu(lz):
    assert lz.device_count() > 0, "GPU tests need a CUDA device (no CPU fallback exists)"
    return lz


def run_capture(lz, w, thr, root, spec_dir, **knobs):
    spec = w.write_spec(os.path.join(spec_dir, w.name + ".spec"))
    built = lz.build_workload(spec, 0)
    knobs = dict(knobs)
    pool = knobs.pop("host_buffer_bytes", max(2 * built.bytes, 1 << 20) + (8 << 20))
    knobs.setdefault("fsync_on_finalize", False)
    cfg = lz.EngineConfig(checkpoint_root=str(root), host_buffer_bytes=pool,
                          large_leaf_threshold=thr, **knobs)
    eng = lz.Engine(cfg, built.topo, built.rank)
    t = eng.capture(lz.plan_checkpoint(built.topo, built.model, built.step), built.tree, built.step)
    eng.update_barrier(t)
    eng.wait_persisted(t)
    assert t.status() == "persisted" and not t.torn()
    return eng, built, t


@pytest.mark.parametrize("variant", list(VARIANTS))
def test_files_match_reference_and_oracle(gpu, oracle, cases, fixtures, tmp_path, variant):
    lz = gpu
    for name, (w, thr) in cases.items():
        root = tmp_path / f"{name}-{variant}"
        eng, built, t = run_capture(lz, w, thr, root, str(tmp_path), **VARIANTS[variant])
        want = fixtures[name]["files"]
        expect = oracle.compose_files(w, thr)
        got = {os.path.relpath(f, root): f for f in t.shard_files()}
        assert set(got) == set(want) == set(expect), name
        assert t.payload_bytes() == fixtures[name]["payload"]
        for rel, path in got.items():
            data = np.fromfile(path, dtype=np.uint8)
            assert data.size == want[rel]["size"], (name, rel)
            assert f"{oracle.fnv64(data):016x}" == want[rel]["fnv"], (name, rel)
            assert np.array_equal(data, expect[rel]), (name, rel)
        eng.close()
        shutil.rmtree(root, ignore_errors=True)


@pytest.mark.parametrize("variant", ["default", "kernel-only", "copy-engine-only"])
def test_many_small_leaves_submitted_in_chunks(gpu, oracle, tmp_path, variant):
    """3000 x 4 KiB leaves, all above the threshold: one file's tasks are
    submitted in chunks of 1024 while the rest are built (engine.cpp); the
    file must still equal the oracle's composition and the ticket's device
    time must span all chunks."""
    lz = gpu
    from paper_2406_10707_b200.workloads import sweep_class
    w = sweep_class(4096, 3000 * 4096)
    eng, built, t = run_capture(lz, w, 4096, tmp_path / "many", str(tmp_path), **VARIANTS[variant])
    expect = oracle.compose_files(w, 4096)
    got = {os.path.relpath(f, tmp_path / "many"): f for f in t.shard_files()}
    assert set(got) == set(expect)
    for rel, path in got.items():
        assert np.array_equal(np.fromfile(path, dtype=np.uint8), expect[rel]), rel
    assert eng.ticket_device_ms(t) > 0
    eng.close()


def test_c1_golden_digests_and_restore(gpu, oracle, tmp_path):
    lz = gpu
    from paper_2406_10707_b200.workloads import gpt2_small
    w = gpt2_small()
    eng, built, t = run_capture(lz, w, 1 << 20, tmp_path / "c1", str(tmp_path))
    got = {}
    for f in t.shard_files():
        data = np.fromfile(f, dtype=np.uint8)
        got[os.path.relpath(f, tmp_path / "c1")] = (data.size, oracle.fnv64(data))
    assert got == C1_GOLDEN
    m = lz.ManifestStore(tmp_path / "c1" / "manifest.json")
    m.commit_step(1, lz.committed_record(t, str(tmp_path / "c1")))
    back = eng.restore(m, 1)
    src = oracle.generate(w)
    index = {p: i for i, (_, p, _) in enumerate(w.leaves)}
    assert back.leaf_count() == len(w.leaves)
    for leaf in back.flatten():
        assert leaf.is_region
        assert back.region_at(leaf.path).clone_bytes() == src[index[leaf.path]].tobytes(), leaf.path
        assert back.region_at(leaf.path).version() == 0
    with pytest.raises(lz.NotCommitted):
        eng.restore(m, 99)
    eng.close()
    shutil.rmtree(tmp_path, ignore_errors=True)


# ---------------------------------------------------------------------------
# kernels through lzk_cuda.h


class Dev:
    def __init__(self, lz):
        self.d = lz.dev

    def ck(self, rc):
        if rc != 0:
            raise RuntimeError(self.d.lzk_last_error().decode())

    def pinned(self, n):
        p = C.c_void_p()
        self.ck(self.d.lzk_host_alloc(max(n, 1), 1, C.byref(p)))
        arr = np.ctypeslib.as_array((C.c_uint8 * max(n, 1)).from_address(p.value))
        return p.value, arr

    def dalloc(self, n):
        p = C.c_void_p()
        self.ck(self.d.lzk_dev_alloc(0, max(n, 1), C.byref(p)))
        return p.value

    def stream(self):
        s = C.c_void_p()
        self.ck(self.d.lzk_stream_create(0, 0, C.byref(s)))
        return s


def descs(items):
    from paper_2406_10707_b200 import _native as N
    arr = (N.CopyDescC * max(len(items), 1))()
    for i, (s, d, n) in enumerate(items):
        arr[i] = N.CopyDescC(s, d, n)
    return arr


@pytest.mark.parametrize("direction", ["d2h", "h2d", "d2d"])
def test_gather_kernel_random_layouts(gpu, direction):
    dv = Dev(gpu)
    rng = np.random.default_rng(17)
    src_bytes = 24 << 20
    dst_bytes = 112 << 20
    host_src_p, host_src = dv.pinned(src_bytes)
    host_dst_p, host_dst = dv.pinned(dst_bytes)
    dsrc, ddst = dv.dalloc(src_bytes), dv.dalloc(dst_bytes)
    host_src[:] = rng.integers(0, 256, src_bytes, dtype=np.uint8)
    dv.ck(dv.d.lzk_memcpy_h2d(0, dsrc, host_src_p, src_bytes))
    s = dv.stream()
    for trial in range(6):
        n = int(rng.integers(1, 2500))
        sizes = rng.integers(0, 40000, n)
        if trial == 0:
            sizes[:5] = [0, 1, 15, 16, 17]
        if trial == 5:
            sizes = rng.integers(200_000, 2_000_000, 8)
            n = len(sizes)
        # non-overlapping destinations at arbitrary byte offsets; sources anywhere
        gaps = rng.integers(0, 40, n)
        doff = np.cumsum(gaps + sizes) - sizes
        assert doff[-1] + sizes[-1] <= dst_bytes
        soff = [int(rng.integers(0, src_bytes - z)) if z < src_bytes else 0 for z in sizes]
        expect = np.zeros(dst_bytes, dtype=np.uint8)
        expect[:] = 0xA5
        ref_src = host_src
        for z, so, do in zip(sizes, soff, doff):
            expect[do:do + z] = ref_src[so:so + z]
        if direction == "d2h":
            host_dst[:] = 0xA5
            arr = descs([(dsrc + so, host_dst_p + int(do), int(z)) for z, so, do in zip(sizes, soff, doff)])
            dv.ck(dv.d.lzk_gather_d2h(s, arr, n, int(rng.integers(0, 20))))
            dv.ck(dv.d.lzk_stream_sync(s))
            got = host_dst
        elif direction == "h2d":
            dv.ck(dv.d.lzk_dev_memset(0, ddst, 0xA5, dst_bytes))
            arr = descs([(host_src_p + so, ddst + int(do), int(z)) for z, so, do in zip(sizes, soff, doff)])
            dv.ck(dv.d.lzk_scatter_h2d(s, arr, n, 0))
            dv.ck(dv.d.lzk_stream_sync(s))
            dv.ck(dv.d.lzk_memcpy_d2h(0, host_dst_p, ddst, dst_bytes))
            got = host_dst
        else:
            dv.ck(dv.d.lzk_dev_memset(0, ddst, 0xA5, dst_bytes))
            arr = descs([(dsrc + so, ddst + int(do), int(z)) for z, so, do in zip(sizes, soff, doff)])
            dv.ck(dv.d.lzk_gather_d2d(s, arr, n, 0))
            dv.ck(dv.d.lzk_stream_sync(s))
            dv.ck(dv.d.lzk_memcpy_d2h(0, host_dst_p, ddst, dst_bytes))
            got = host_dst
        bad = np.nonzero(got != expect)[0]
        assert bad.size == 0, (direction, trial, bad[:10])
    dv.d.lzk_stream_destroy(s)
    dv.d.lzk_dev_free(0, dsrc)
    dv.d.lzk_dev_free(0, ddst)
    dv.d.lzk_host_free(host_src_p)
    dv.d.lzk_host_free(host_dst_p)


def test_fill_kernel_matches_oracle_generator(gpu, oracle):
    dv = Dev(gpu)
    s = dv.stream()
    for leaf, size in [(0, 1), (3, 7), (9, 8), (12, 4097), (77, 1 << 20)]:
        d = dv.dalloc(size)
        dv.ck(dv.d.lzk_fill_splitmix(s, d, size, 1234, leaf))
        dv.ck(dv.d.lzk_stream_sync(s))
        p, h = dv.pinned(size)
        dv.ck(dv.d.lzk_memcpy_d2h(0, p, d, size))
        want = np.empty(size, dtype=np.uint8)
        oracle.L.lzo_fill_splitmix(1234, leaf, size, want.ctypes.data)
        assert np.array_equal(h[:size], want)
        dv.d.lzk_host_free(p)
        dv.d.lzk_dev_free(0, d)
    dv.d.lzk_stream_destroy(s)


# ---------------------------------------------------------------------------
# lazy fence semantics


def small_engine(lz, root, **kw):
    topo = lz.ParallelTopology(1, 1, 1, 1, 1)
    cfg = lz.EngineConfig(checkpoint_root=str(root), host_buffer_bytes=64 << 20, large_leaf_threshold=4096,
                          fsync_on_finalize=False, **kw)
    return lz.Engine(cfg, topo, lz.RankCoord()), topo


def tiny_model(lz):
    return lz.ModelSpec(param_count=4096, layer_count=4)


def mixed_tree(lz, rng):
    t = lz.StateTree()
    regs = {}
    for path, n in [("layers/block0/w", 5000), ("layers/block1/w", 3192), ("optim/moments", 40000)]:
        regs[path] = lz.DeviceRegion(rng.integers(0, 256, n, dtype=np.uint8).tobytes())
        t.set_region(path, regs[path])
    t.set_blob("optim/step", b"\x01" * 8)
    t.set_blob("optim/extra", bytes(9144))
    return t, regs


def test_mutation_mid_copy_tears_and_files_stay_headerless(gpu, tmp_path):
    """reference test_engine.cpp:183-215 through the Python/C ABI: a paced
    channel (50 MB/s), the first shard's region mutated before the barrier."""
    lz = gpu
    topo = lz.ParallelTopology(1, 1, 1, 1, 1)
    cfg = lz.EngineConfig(checkpoint_root=str(tmp_path), host_buffer_bytes=32 << 20, large_leaf_threshold=4096,
                          fsync_on_finalize=False, copy_bandwidth_Bps=50e6, chunk_quantum=64 << 10)
    eng = lz.Engine(cfg, topo, lz.RankCoord())
    model = lz.ModelSpec(param_count=1 << 20, layer_count=4)
    weights = lz.DeviceRegion(bytes(range(256)) * (8192))  # 2 MiB
    tree = lz.StateTree()
    tree.set_region("layers/w", weights)
    tree.set_region("optim/m", lz.DeviceRegion(12 << 20))
    t = eng.capture(lz.plan_checkpoint(topo, model, 5), tree, 5)
    time.sleep(0.005)
    weights.write(0, b"\x01")
    with pytest.raises(lz.TornSnapshot):
        eng.update_barrier(t)
    assert t.torn() and t.status() == "failed" and "changed" in t.failure_reason()
    with pytest.raises(lz.TornSnapshot):
        eng.wait_persisted(t)
    eng.drain()
    for f in t.shard_files():
        assert os.path.exists(f)
        with pytest.raises(lz.BadMagic):
            lz.read_header(f)
    eng.close()


def test_unpaced_mutation_after_barrier_is_not_torn(gpu, tmp_path):
    lz = gpu
    rng = np.random.default_rng(2)
    eng, topo = small_engine(lz, tmp_path)
    tree, regs = mixed_tree(lz, rng)
    before = {p: r.clone_bytes() for p, r in regs.items()}
    t = eng.capture(lz.plan_checkpoint(topo, tiny_model(lz), 6), tree, 6)
    eng.update_barrier(t)
    regs["optim/moments"].mutate(lambda b: b.__setitem__(slice(0, 100), bytes(100)))
    eng.wait_persisted(t)
    assert not t.torn()
    h = lz.read_header(t.shard_files()[1])
    assert lz.read_entry(t.shard_files()[1], h, "optim/moments") == before["optim/moments"]
    eng.close()


def test_small_leaves_are_captured_at_capture_time(gpu, tmp_path):
    """reference test_engine.cpp:217-240: inline leaves are snapshotted
    synchronously, so a mutation right after capture() cannot reach them."""
    lz = gpu
    eng, topo = small_engine(lz, tmp_path, copy_bandwidth_Bps=5e6, chunk_quantum=4096)
    t_ = lz.StateTree()
    small = lz.DeviceRegion(bytes(range(256)) * 4)  # 1024 B < threshold
    big = lz.DeviceRegion(bytes(8192 - 1024))
    t_.set_region("layers/small", small)
    t_.set_region("layers/big", big)
    t_.set_region("optim/m", lz.DeviceRegion(bytes(49152)))
    t = eng.capture(lz.plan_checkpoint(topo, tiny_model(lz), 7), t_, 7)
    small.write(0, b"\xff" * 16)  # after capture, before barrier
    eng.update_barrier(t)
    eng.wait_persisted(t)
    m = lz.ManifestStore(tmp_path / "manifest.json")
    m.commit_step(7, lz.committed_record(t, str(tmp_path)))
    back = eng.restore(m, 7)
    assert back.region_at("layers/small").clone_bytes() == bytes(range(256)) * 4
    eng.close()


def test_device_side_fence_orders_optimizer_after_snapshot(gpu, tmp_path):
    """update_barrier_on_stream: the trainer's stream waits for the snapshot;
    the 'optimizer step' queued after it must not leak into the checkpoint,
    and the declared mutation (bump_version) after the fence is not a tear."""
    lz = gpu
    torch = pytest.importorskip("torch")
    eng, topo = small_engine(lz, tmp_path)
    layers = torch.arange(2048, dtype=torch.float32, device="cuda")  # 8192 B
    optim = torch.full((12288,), 3.0, dtype=torch.float32, device="cuda")  # 49152 B
    torch.cuda.synchronize()
    tree = lz.StateTree()
    rl, ro = lz.DeviceRegion.wrap(layers), lz.DeviceRegion.wrap(optim)
    tree.set_region("layers/w", rl)
    tree.set_region("optim/m", ro)
    want = optim.cpu().numpy().tobytes()
    s = torch.cuda.Stream()
    for step in range(1, 4):
        t = eng.capture(lz.plan_checkpoint(topo, tiny_model(lz), step), tree, step)
        eng.update_barrier_on_stream(t, s.cuda_stream)
        with torch.cuda.stream(s):
            optim.add_(1.0)  # optimizer step, stream-ordered after the snapshot
        ro.bump_version()
        eng.wait_persisted(t)
        assert not t.torn()
        f = t.shard_files()[1]
        got = lz.read_entry(f, lz.read_header(f), "optim/m")
        assert got == want, step
        s.synchronize()
        want = optim.cpu().numpy().tobytes()
    eng.close()


def test_restore_into_existing_regions(gpu, tmp_path):
    lz = gpu
    rng = np.random.default_rng(4)
    eng, topo = small_engine(lz, tmp_path)
    tree, regs = mixed_tree(lz, rng)
    before = {p: r.clone_bytes() for p, r in regs.items()}
    t = eng.capture(lz.plan_checkpoint(topo, tiny_model(lz), 9), tree, 9)
    eng.update_barrier(t)
    eng.wait_persisted(t)
    m = lz.ManifestStore(tmp_path / "manifest.json")
    m.commit_step(9, lz.committed_record(t, str(tmp_path)))
    for r in regs.values():
        r.write(0, b"\x00" * 64)
    v = regs["optim/moments"].version()
    eng.restore_into(m, 9, tree)
    for p, r in regs.items():
        assert r.clone_bytes() == before[p]
    assert regs["optim/moments"].version() > v
    eng.close()


def test_corrupt_file_is_rejected_on_restore(gpu, tmp_path):
    lz = gpu
    rng = np.random.default_rng(5)
    eng, topo = small_engine(lz, tmp_path)
    tree, _ = mixed_tree(lz, rng)
    t = eng.capture(lz.plan_checkpoint(topo, tiny_model(lz), 3), tree, 3)
    eng.update_barrier(t)
    eng.wait_persisted(t)
    m = lz.ManifestStore(tmp_path / "manifest.json")
    m.commit_step(3, lz.committed_record(t, str(tmp_path)))
    f = t.shard_files()[1]
    raw = bytearray(open(f, "rb").read())
    raw[-5] ^= 0x40
    open(f, "wb").write(raw)
    with pytest.raises(lz.ChecksumMismatch):
        eng.restore(m, 3)
    open(f, "wb").write(raw[:-1])
    with pytest.raises(lz.TruncatedFile):
        eng.restore(m, 3)
    eng.close()


def test_pool_backpressure_blocks_capture_until_flush_releases(gpu, tmp_path):
    lz = gpu
    rng = np.random.default_rng(6)
    topo = lz.ParallelTopology(1, 1, 1, 1, 1)
    # pool fits one capture (~57.5 KB payload) but not two; slow storage
    cfg = lz.EngineConfig(checkpoint_root=str(tmp_path), host_buffer_bytes=80_000, large_leaf_threshold=4096,
                          fsync_on_finalize=False, storage_bandwidth_Bps=1e6)
    eng = lz.Engine(cfg, topo, lz.RankCoord())
    tree, _ = mixed_tree(lz, rng)
    t1 = eng.capture(lz.plan_checkpoint(topo, tiny_model(lz), 1), tree, 1)
    eng.update_barrier(t1)
    t0 = time.perf_counter()
    t2 = eng.capture(lz.plan_checkpoint(topo, tiny_model(lz), 2), tree, 2)
    waited = time.perf_counter() - t0
    assert waited > 0.02  # blocked on t1's flush (57 KB at 1 MB/s)
    eng.update_barrier(t2)
    eng.wait_persisted(t2)
    assert t1.status() == "persisted" and t2.status() == "persisted"
    with pytest.raises(lz.SizeExceedsCapacity):
        big = lz.StateTree()
        big.set_region("layers/w", lz.DeviceRegion(8192))
        big.set_region("optim/m", lz.DeviceRegion(49152))
        small_cfg = lz.EngineConfig(checkpoint_root=str(tmp_path / "x"), host_buffer_bytes=40_000,
                                    large_leaf_threshold=4096)
        e2 = lz.Engine(small_cfg, topo, lz.RankCoord())
        e2.capture(lz.plan_checkpoint(topo, tiny_model(lz), 1), big, 1)
    eng.close()


def test_streaming_c1_through_a_small_pool(gpu, oracle, tmp_path):
    """C1 (1.74 GB) through a 256 MB pool in 48 MB segments: golden digests,
    capture never blocks, the fence waits for the storage tier."""
    lz = gpu
    from paper_2406_10707_b200.workloads import gpt2_small
    w = gpt2_small()
    spec = w.write_spec(str(tmp_path / "c1.spec"))
    built = lz.build_workload(spec, 0)
    root = tmp_path / "c1s"
    cfg = lz.EngineConfig(checkpoint_root=str(root), host_buffer_bytes=256 << 20, stream_segment_bytes=48 << 20,
                          fsync_on_finalize=False)
    eng = lz.Engine(cfg, built.topo, built.rank)
    t0 = time.perf_counter()
    t = eng.capture(lz.plan_checkpoint(built.topo, built.model, 1), built.tree, 1)
    assert time.perf_counter() - t0 < 1.0  # no wait for the 1.7 GB to drain
    eng.update_barrier(t)
    eng.wait_persisted(t)
    got = {}
    for f in t.shard_files():
        data = np.fromfile(f, dtype=np.uint8)
        got[os.path.relpath(f, root)] = (data.size, oracle.fnv64(data))
    assert got == C1_GOLDEN
    eng.close()
    shutil.rmtree(tmp_path, ignore_errors=True)


@pytest.mark.parametrize("variant", ["kernel", "copy_engine"])
def test_tensor_larger_than_4gib_misaligned(gpu, tmp_path, variant):
    """A 4.5 GiB + 7 B leaf after a 13 B meta-sized offset: 64-bit sizes and
    offsets through the gather kernel and the DMA path, checked by sampled
    windows (head, 4 GiB boundary, tail) against the device bytes."""
    lz = gpu
    torch = pytest.importorskip("torch")
    n = (9 << 29) + 7
    big = torch.empty(n, dtype=torch.uint8, device="cuda")
    d = lz.dev
    import ctypes as C
    s = C.c_void_p()
    assert d.lzk_stream_create(0, 0, C.byref(s)) == 0
    assert d.lzk_fill_splitmix(s, big.data_ptr(), n, 99, 3) == 0
    assert d.lzk_stream_sync(s) == 0
    d.lzk_stream_destroy(s)
    topo = lz.ParallelTopology(1, 1, 1, 1, 1)
    params = (n + 13) // 2  # layer shard = 2 B/param; a 1 B/param optimizer keeps the files small
    model = lz.ModelSpec(param_count=params, layer_count=1, bytes_per_param_optimizer=1)
    plan = lz.plan_checkpoint(topo, model, 1)
    layer_bytes, opt_bytes = [x.size_bytes for x in plan.shards(0)]
    tree = lz.StateTree()
    tree.set_region("a/big", lz.DeviceRegion.wrap(big))
    tree.set_blob("a/pad", bytes(layer_bytes - n))
    opt = torch.zeros(opt_bytes, dtype=torch.uint8, device="cuda")
    tree.set_region("b/o", lz.DeviceRegion.wrap(opt))
    cfg = lz.EngineConfig(checkpoint_root=str(tmp_path), host_buffer_bytes=layer_bytes + opt_bytes + (64 << 20),
                          fsync_on_finalize=False, large_leaf_threshold=1 << 20,
                          force_kernel=variant == "kernel", force_copy_engine=variant == "copy_engine")
    eng = lz.Engine(cfg, topo, lz.RankCoord())
    t = eng.capture(plan, tree, 1)
    eng.update_barrier(t)
    eng.wait_persisted(t)
    f = [p for p in t.shard_files() if "layers" in p][0]
    h = lz.read_header(f)
    e = h.find("a/big")
    assert e.length == n
    with open(f, "rb") as fh:
        for off in (0, (1 << 32) - 4096, n - 5000):
            fh.seek(e.offset + off)
            got = fh.read(5000)
            assert got == big[off:off + 5000].cpu().numpy().tobytes(), off
    assert lz.validate_entries(f, h) == []
    eng.close()
    shutil.rmtree(tmp_path, ignore_errors=True)  # ~7 GB of files: keep the box's disk free


def test_unpaced_mutation_before_barrier_is_torn(gpu, tmp_path):
    """Fast path (device-issued copies): a declared mutation that lands while
    the D2H is still running tears the ticket; no file gets a header."""
    lz = gpu
    torch = pytest.importorskip("torch")
    topo = lz.ParallelTopology(1, 1, 1, 1, 1)
    n = 2 << 30
    model = lz.ModelSpec(param_count=n // 2, layer_count=1, bytes_per_param_optimizer=2)
    plan = lz.plan_checkpoint(topo, model, 1)
    lb, ob = [x.size_bytes for x in plan.shards(0)]
    w = torch.zeros(lb, dtype=torch.uint8, device="cuda")
    o = torch.zeros(ob, dtype=torch.uint8, device="cuda")
    tree = lz.StateTree()
    rw = lz.DeviceRegion.wrap(w)
    tree.set_region("a/w", rw)
    tree.set_region("b/o", lz.DeviceRegion.wrap(o))
    cfg = lz.EngineConfig(checkpoint_root=str(tmp_path), host_buffer_bytes=lb + ob + (64 << 20),
                          fsync_on_finalize=False)
    eng = lz.Engine(cfg, topo, lz.RankCoord())
    t = eng.capture(plan, tree, 1)
    rw.write(0, b"\x01")  # ~80 ms of D2H still ahead (4 GB)
    with pytest.raises(lz.TornSnapshot):
        eng.update_barrier(t)
    with pytest.raises(lz.TornSnapshot):
        eng.wait_persisted(t)
    eng.drain()
    for f in t.shard_files():
        with pytest.raises(lz.BadMagic):
            lz.read_header(f)
    eng.close()
    shutil.rmtree(tmp_path, ignore_errors=True)


def test_rejected_captures_reserve_nothing(gpu, tmp_path):
    """reference test_engine.cpp:141-170: a plan/tree mismatch or the reserved
    metadata name throws before any pool space is taken."""
    lz = gpu
    eng, topo = small_engine(lz, tmp_path)
    plan = lz.plan_checkpoint(topo, tiny_model(lz), 1)
    one = lz.StateTree()
    one.set_region("layers/w", lz.DeviceRegion(8192))
    with pytest.raises(lz.ConfigError):  # one child, two shards
        eng.capture(plan, one, 1)
    wrong = lz.StateTree()
    wrong.set_region("layers/w", lz.DeviceRegion(8000))
    wrong.set_region("optim/m", lz.DeviceRegion(49152))
    with pytest.raises(lz.ConfigError):  # sizes do not match the plan
        eng.capture(plan, wrong, 1)
    meta = lz.StateTree()
    meta.set_region("__meta__", lz.DeviceRegion(8192))
    meta.set_region("optim/m", lz.DeviceRegion(49152))
    with pytest.raises(lz.DuplicatePath):
        eng.capture(plan, meta, 1)
    assert eng.counters().captures == 0
    ok = lz.StateTree()
    ok.set_region("layers/w", lz.DeviceRegion(8192))
    ok.set_region("optim/m", lz.DeviceRegion(49152))
    t = eng.capture(plan, ok, 1)  # the pool is still whole
    eng.update_barrier(t)
    eng.wait_persisted(t)
    assert t.status() == "persisted"
    eng.close()


def test_deepspeed_style_checkpoint_engine_roundtrip(gpu, tmp_path):
    """Framework glue: a torch model + Adam state saved through the
    DeepSpeed-style engine while training continues after wait(); load()
    returns exactly the snapshot taken at save time (all dtypes, CPU tensors,
    non-contiguous views, scalars, nested containers)."""
    torch = pytest.importorskip("torch")
    from paper_2406_10707_b200.checkpoint_engine import DataStatesCheckpointEngine
    torch.manual_seed(0)
    model = torch.nn.Sequential(torch.nn.Linear(512, 1024), torch.nn.GELU(), torch.nn.Linear(1024, 256)).cuda()
    model[2].to(torch.bfloat16)
    opt = torch.optim.Adam(model.parameters(), lr=1e-3)
    for _ in range(2):
        x = torch.randn(64, 512, device="cuda")
        out = model[2](model[1](model[0](x)).to(torch.bfloat16))
        out.float().pow(2).mean().backward()
        opt.step()
        opt.zero_grad()
    extra = {"step": 7, "lr": [1e-3, 2e-4], "cpu_buf": torch.arange(10, dtype=torch.int64),
             "view": torch.randn(32, 64, device="cuda").t(), "empty": torch.empty(0, device="cuda"),
             "scalar": torch.tensor(3.5, device="cuda"), ("tuple", "key"): None}
    state = {"module": model.state_dict(), "optimizer": opt.state_dict(), "extra": extra}
    expect = {k: v.detach().clone().cpu() for k, v in model.state_dict().items()}
    expect_opt = {k: {n: (t.detach().clone().cpu() if torch.is_tensor(t) else t) for n, t in st.items()}
                  for k, st in opt.state_dict()["state"].items()}
    eng = DataStatesCheckpointEngine({"datastates_ckpt": {"host_cache_size": 64 << 20, "fsync": False}})
    eng.create("global_step7")
    eng.makedirs(str(tmp_path / "global_step7"), exist_ok=True)
    eng.save(state, str(tmp_path / "global_step7" / "mp_rank_00_model_states.pt"))
    eng.wait(torch.cuda.current_stream())  # device-side lazy fence
    x = torch.randn(64, 512, device="cuda")  # training continues: mutates params and Adam state
    model[2](model[1](model[0](x)).to(torch.bfloat16)).float().sum().backward()
    opt.step()
    assert eng.commit("global_step7")
    back = eng.load(str(tmp_path / "global_step7" / "mp_rank_00_model_states.pt"))
    for k, v in expect.items():
        got = back["module"][k]
        assert got.dtype == v.dtype and got.is_cuda and torch.equal(got.cpu(), v), k
    for k, st in expect_opt.items():
        for n, t in st.items():
            g = back["optimizer"]["state"][k][n]
            assert torch.equal(g.cpu(), t) if torch.is_tensor(t) else g == t
    assert back["optimizer"]["param_groups"] == opt.state_dict()["param_groups"]
    e = back["extra"]
    assert e["step"] == 7 and e["lr"] == [1e-3, 2e-4] and e[("tuple", "key")] is None
    assert torch.equal(e["cpu_buf"], extra["cpu_buf"]) and not e["cpu_buf"].is_cuda
    assert torch.equal(e["view"].cpu(), extra["view"].cpu()) and e["view"].shape == (64, 32)
    assert e["empty"].numel() == 0 and float(e["scalar"]) == 3.5
    cpu = eng.load(str(tmp_path / "global_step7" / "mp_rank_00_model_states.pt"), map_location="cpu")
    assert all(not t.is_cuda for t in cpu["module"].values())
    eng.close()


def test_restores_files_written_by_the_reference_engine(gpu, oracle, cases, tmp_path):
    """Cross-implementation: the reference engine (oracle/_ref/ref_snapshot,
    built from the reference sources) writes and commits a checkpoint; our
    engine restores it from the reference's own manifest, byte-exact."""
    import json
    import subprocess
    lz = gpu
    drv = os.path.join(ROOT, "oracle", "_ref", "ref_snapshot")
    assert os.path.exists(drv), "oracle/_ref not built (run __graft_entry__.build() where /root/reference exists)"
    w, thr = cases["odd-sizes"]
    spec = w.write_spec(str(tmp_path / "w.spec"))
    root = tmp_path / "refckpt"
    r = subprocess.run([drv, "--spec", spec, "--root", str(root), "--threshold", str(thr), "--restore", "1"],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert json.loads(r.stdout)["ranks"][0]["restore_exact"]
    topo = lz.ParallelTopology(*w.topology)
    cfg = lz.EngineConfig(checkpoint_root=str(root), host_buffer_bytes=64 << 20, large_leaf_threshold=thr)
    eng = lz.Engine(cfg, topo, lz.RankCoord(*w.rank))
    m = lz.ManifestStore(root / "manifest-0.json")
    back = eng.restore(m, w.step)
    src = oracle.generate(w)
    for i, (kind, path, _) in enumerate(w.leaves):
        got = back.region_at(path).clone_bytes() if kind == "r" else back.blob_at(path)
        assert got == src[i].tobytes(), path
    eng.close()


def test_restore_and_commit_entries_spanning_windows(gpu, oracle, tmp_path):
    """Entries larger than the 512 MiB restore window (continued device
    digests across windows, D2D scatter of window slices): a 1.2 GB and an
    odd-sized ~700 MB region plus small ones, persisted, committed (GPU
    validation), restored fresh and in place; restored bytes compared with
    the sources by device FNV-1a (lz.device_fnv64, bit-exact vs the oracle in
    test_gpu_fnv.py)."""
    import ctypes as Cc
    lz = gpu
    sizes = {"big/w": (1200 << 20) + 3, "big/x": (700 << 20) - 13, "small/a": 4097, "small/b": 1 << 20}
    tree = lz.StateTree()
    regs = {}
    s = Cc.c_void_p()
    assert lz.dev.lzk_stream_create(0, 0, Cc.byref(s)) == 0
    for i, (path, n) in enumerate(sizes.items()):
        r = lz.DeviceRegion(n)
        assert lz.dev.lzk_fill_splitmix(s, r.device_ptr, n, 77, i) == 0
        regs[path] = r
        tree.set_region(path, r)
    assert lz.dev.lzk_stream_sync(s) == 0
    lz.dev.lzk_stream_destroy(s)
    want = dict(zip(sizes, lz.device_fnv64([(regs[p].device_ptr, n) for p, n in sizes.items()])))
    total = sum(sizes.values())
    topo = lz.ParallelTopology(1, 1, 1, 1, 1)
    cfg = lz.EngineConfig(checkpoint_root=str(tmp_path), host_buffer_bytes=total + (256 << 20),
                          large_leaf_threshold=1 << 20, fsync_on_finalize=False)
    eng = lz.Engine(cfg, topo, lz.RankCoord())
    t = eng.capture_file(str(tmp_path / "span.ckpt"), tree, 1)
    eng.wait_persisted(t)
    back = eng.restore_file(str(tmp_path / "span.ckpt"))
    got = dict(zip(sizes, lz.device_fnv64([(back.region_at(p).device_ptr, n) for p, n in sizes.items()])))
    assert got == want
    del back
    # in place: clobber the live regions, restore into them
    for p, r in regs.items():
        assert lz.dev.lzk_dev_memset(0, r.device_ptr, 0, sizes[p]) == 0
    eng.restore_file(str(tmp_path / "span.ckpt"), into=tree)
    got = dict(zip(sizes, lz.device_fnv64([(regs[p].device_ptr, n) for p, n in sizes.items()])))
    assert got == want
    # whole-file digest on the GPU (windows continued) == the oracle's fold
    (rel, n, d), = lz.committed_record(t, str(tmp_path), digest=True)
    assert n == os.path.getsize(tmp_path / "span.ckpt")
    assert d == oracle.fnv64(np.fromfile(tmp_path / "span.ckpt", dtype=np.uint8))
    eng.close()


def test_engine_ring_on_the_gpu_numa_node(gpu, tmp_path):
    """the pinned ring (and the engine threads) sit on the
    GPU's NUMA node; on single-node hosts the placement is a no-op (-1)."""
    lz = gpu
    eng, _ = small_engine(lz, tmp_path)
    dev_node = lz.device_numa_node(0)
    if lz.numa_node_count() < 2 or dev_node < 0:
        assert eng.numa_node() == -1
    else:
        assert eng.numa_node() == dev_node
    eng.close()


def test_restore_file_into_live_regions_validates_first(gpu, tmp_path):
    """restore_file(path, into): a corrupt file raises ChecksumMismatch and
    leaves the caller's live regions untouched (every entry is validated
    before the first byte lands in them, as restore_into does)."""
    lz = gpu
    eng, _ = small_engine(lz, tmp_path)
    tree = lz.StateTree()
    tree.set_region("x/big", lz.DeviceRegion(bytes(range(256)) * 64))  # 16 KiB: a payload entry
    tree.set_region("x/small", lz.DeviceRegion(b"abc" * 10))            # inline in __meta__
    f = tmp_path / "one.lzckpt"
    t = eng.capture_file(str(f), tree, 1)
    eng.update_barrier(t)
    eng.wait_persisted(t)
    raw = bytearray(f.read_bytes())
    raw[-5] ^= 0xFF  # inside x/big, the last payload entry
    f.write_bytes(bytes(raw))
    live = lz.StateTree()
    target = lz.DeviceRegion(bytes(16384))
    live.set_region("x/big", target)
    live.set_region("x/small", lz.DeviceRegion(bytes(30)))
    with pytest.raises(lz.ChecksumMismatch):
        eng.restore_file(str(f), live)
    assert target.clone_bytes() == bytes(16384)
    eng.close()
