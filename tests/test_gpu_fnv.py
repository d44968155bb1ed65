"""Device FNV-1a-64 (lzk_fnv1a64_batch, paper_2406_10707_b200/csrc/cuda/lzk_fnv.cu)
against the oracle's byte-serial fold (oracle/lzk_oracle.c lzo_fnv1a64, which
follows the reference's include/lzckpt/checksum.hpp:17-24). Bit-exact: these
are integer digests. Covers every length class of the kernel (aligned head,
full 1 KiB warp windows, partial window), arbitrary source alignment,
continued states (non-basis seeds), both output kinds (mapped host and device
memory), multi-launch batches and GB-scale entries."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

BASIS = 0xCBF29CE484222325


@pytest.fixture(scope="module")
def gpu(lz):
    assert lz.device_count() > 0, "GPU tests need a CUDA device (no CPU fallback exists)"
    return lz


class Buf:
    """Random bytes resident in HBM (and a host copy for the oracle)."""

    def __init__(self, lz, n, seed):
        self.lz = lz
        self.host = np.random.default_rng(seed).integers(0, 256, n, dtype=np.uint8)
        p = C.c_void_p()
        assert lz.dev.lzk_dev_alloc(0, n, C.byref(p)) == 0
        self.ptr = p.value
        assert lz.dev.lzk_memcpy_h2d(0, self.ptr, self.host.ctypes.data, n) == 0

    def free(self):
        self.lz.dev.lzk_dev_free(0, self.ptr)


def test_fnv_lengths_alignments_seeds(gpu, oracle):
    buf = Buf(gpu, 8 << 20, 1)
    rng = np.random.default_rng(2)
    lens = [0, 1, 2, 15, 16, 17, 31, 32, 33, 63, 1023, 1024, 1025, 1039, 2047, 2048, 3072 + 5, 4096, 65543,
            (1 << 20) + 13]
    lens += [int(x) for x in rng.integers(0, 200_000, 300)]
    ranges, seeds, want = [], [], []
    for i, n in enumerate(lens):
        off = int(rng.integers(0, (8 << 20) - n)) if i % 3 else int(rng.integers(0, 64)) * 16
        seed = BASIS if i % 2 == 0 else int(rng.integers(0, 1 << 63)) * 2 + (i & 1)
        ranges.append((buf.ptr + off, n))
        seeds.append(seed)
        want.append(oracle.fnv64(buf.host[off:off + n], seed))
    for ctas in (0, 1, 3):
        got = gpu.device_fnv64(ranges, seeds=seeds, max_ctas=ctas)
        bad = [(i, lens[i]) for i in range(len(lens)) if got[i] != want[i]]
        assert not bad, (ctas, bad[:10])
    buf.free()


def test_fnv_device_output_and_multilaunch(gpu, oracle):
    """> 960 ranges (several launches) with results stored to HBM."""
    from paper_2406_10707_b200 import _native as N
    buf = Buf(gpu, 4 << 20, 3)
    rng = np.random.default_rng(4)
    n = 2500
    lens = rng.integers(0, 5000, n)
    offs = [int(rng.integers(0, (4 << 20) - int(z))) for z in lens]
    out = C.c_void_p()
    assert gpu.dev.lzk_dev_alloc(0, 8 * n, C.byref(out)) == 0
    arr = (N.HashDescC * n)()
    for i in range(n):
        arr[i] = N.HashDescC(buf.ptr + offs[i], int(lens[i]), BASIS, out.value + 8 * i)
    s = C.c_void_p()
    assert gpu.dev.lzk_stream_create(0, 0, C.byref(s)) == 0
    assert gpu.dev.lzk_fnv1a64_batch(s, arr, n, 0) == 0
    assert gpu.dev.lzk_stream_sync(s) == 0
    got = np.zeros(n, dtype=np.uint64)
    assert gpu.dev.lzk_memcpy_d2h(0, got.ctypes.data, out.value, 8 * n) == 0
    for i in range(n):
        assert int(got[i]) == oracle.fnv64(buf.host[offs[i]:offs[i] + int(lens[i])]), i
    gpu.dev.lzk_stream_destroy(s)
    gpu.dev.lzk_dev_free(0, out)
    buf.free()


def test_fnv_rejects_bad_descriptors(gpu):
    from paper_2406_10707_b200 import _native as N
    arr = (N.HashDescC * 1)(N.HashDescC(0x1000, 16, BASIS, 0))
    s = C.c_void_p()
    assert gpu.dev.lzk_stream_create(0, 0, C.byref(s)) == 0
    assert gpu.dev.lzk_fnv1a64_batch(s, arr, 1, 0) == 1  # null output
    arr[0] = N.HashDescC(0, 16, BASIS, 0x1000)
    assert gpu.dev.lzk_fnv1a64_batch(s, arr, 1, 0) == 1  # null source
    gpu.dev.lzk_stream_destroy(s)


def test_fnv_gb_scale_entries(gpu, oracle):
    """Long single-warp chains: 2 x 384 MiB at odd offsets, checked against
    the oracle fold; and the splitmix64 generator's digest of a 1 GiB leaf
    (oracle lzo_splitmix_fnv: no host copy needed)."""
    n = 384 << 20
    buf = Buf(gpu, 2 * n + 64, 5)
    ranges = [(buf.ptr + 3, n), (buf.ptr + n + 40, n - 7)]
    want = [oracle.fnv64(buf.host[3:3 + n]), oracle.fnv64(buf.host[n + 40:2 * n + 33])]
    assert gpu.device_fnv64(ranges) == want
    buf.free()
    size = (1 << 30) + 5
    p = C.c_void_p()
    assert gpu.dev.lzk_dev_alloc(0, size, C.byref(p)) == 0
    s = C.c_void_p()
    assert gpu.dev.lzk_stream_create(0, 0, C.byref(s)) == 0
    assert gpu.dev.lzk_fill_splitmix(s, p.value, size, 99, 7) == 0
    assert gpu.dev.lzk_stream_sync(s) == 0
    assert gpu.device_fnv64([(p.value, size)]) == [oracle.L.lzo_splitmix_fnv(99, 7, size)]
    gpu.dev.lzk_stream_destroy(s)
    gpu.dev.lzk_dev_free(0, p.value)


def test_fnv_segmented_long_ranges(gpu, oracle):
    """Ranges larger than a fair share of the grid take the multi-pass
    segmented schedule (8 plane passes + final + combine): odd offsets and
    lengths, non-basis seeds, mixed with short ranges in one batch."""
    buf = Buf(gpu, 96 << 20, 6)
    rng = np.random.default_rng(7)
    items = [(3, (4 << 20) + 5), (1 << 20, (9 << 20) + 1023), (17 << 20, (33 << 20) + 7), (80 << 20, 1000),
             (81 << 20, (5 << 20) - 1), (90 << 20, 12345)]
    seeds = [int(rng.integers(0, 1 << 62)) for _ in items]
    want = [oracle.fnv64(buf.host[o:o + n], sd) for (o, n), sd in zip(items, seeds)]
    for ctas in (0, 4):
        got = gpu.device_fnv64([(buf.ptr + o, n) for o, n in items], seeds=seeds, max_ctas=ctas)
        assert got == want, ctas
    buf.free()


def test_fnv_continue_across_pieces(gpu, oracle):
    """lzk_fnv1a64_continue: a running digest carried in memory across
    launches (restore hashes an entry window by window this way)."""
    from paper_2406_10707_b200 import _native as N
    buf = Buf(gpu, 40 << 20, 8)
    cuts = [0, 7, 1 << 20, (1 << 20) + 3, (30 << 20) + 11, 40 << 20]
    out = C.c_void_p()
    assert gpu.dev.lzk_host_alloc(8, 1, C.byref(out)) == 0
    state = (C.c_uint64 * 1).from_address(out.value)
    state[0] = BASIS
    s = C.c_void_p()
    assert gpu.dev.lzk_stream_create(0, 0, C.byref(s)) == 0
    for a, b in zip(cuts, cuts[1:]):
        arr = (N.HashDescC * 1)(N.HashDescC(buf.ptr + a, b - a, 0, out.value))
        assert gpu.dev.lzk_fnv1a64_continue(s, arr, 1, 0) == 0
    assert gpu.dev.lzk_stream_sync(s) == 0
    assert state[0] == oracle.fnv64(buf.host)
    gpu.dev.lzk_stream_destroy(s)
    gpu.dev.lzk_host_free(out)
    buf.free()
