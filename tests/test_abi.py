"""CPU checks of the drop-in boundary: both C-ABI libraries load and export
every entry point include/*.h declares; the host-side logic behind the C ABI
(ring, header codec, plan, flatten order, manifest, error mapping) agrees
with the oracle; device calls fail loudly without a GPU (no CPU fallback)."""
import ctypes
import os
import random
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared(header):
    txt = open(os.path.join(ROOT, "include", header)).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return set(re.findall(r"\b((?:lzk|lzckpt)_[a-z0-9_]+)\s*\(", txt))


@pytest.mark.parametrize("header,so", [("lzk_cuda.h", "liblzk_cuda.so"), ("lzckpt_c.h", "liblzckpt_b200.so")])
def test_library_exports_every_declared_symbol(header, so):
    lib = ctypes.CDLL(os.path.join(ROOT, "paper_2406_10707_b200", "lib", so))
    names = declared(header)
    assert len(names) > 30
    missing = [n for n in sorted(names) if not hasattr(lib, n)]
    assert not missing, missing


def test_python_bindings_cover_the_headers(lz):
    from paper_2406_10707_b200 import _native as N
    bound = {n for n, _, _ in N.ENGINE_SYMBOLS} | {n for n, _, _ in N.DEVICE_SYMBOLS}
    assert declared("lzckpt_c.h") <= bound
    assert declared("lzk_cuda.h") <= bound


def test_fnv_matches_oracle(lz, oracle):
    rng = random.Random(3)
    for n in (0, 1, 7, 8, 9, 1000, 65537):
        data = bytes(rng.getrandbits(8) for _ in range(n))
        assert lz.fnv64(data) == oracle.fnv64(data)


def test_ring_matches_oracle_randomized(lz, oracle):
    """reference tests/test_ring.cpp:196-261 style: random op sequences."""
    rng = random.Random(7)
    for trial in range(200):
        cap = rng.randint(1, 5000)
        a, b = lz.RingCore(cap), oracle.Ring(cap)
        live = []  # FIFO of (id, state)
        for _ in range(60):
            op = rng.random()
            if op < 0.5:
                size = rng.randint(0, cap + 2)
                ra, rb = a.try_reserve(size, 1), b.try_reserve(size)
                assert ra == rb, (trial, size)
                if ra:
                    live.append([ra[0], 0])
            elif live:
                sid, st = live[0] if op < 0.8 else rng.choice(live)
                if st == 0:
                    a.mark_filled(sid), b.mark_filled(sid)
                elif st == 1:
                    a.begin_flush(sid), b.begin_flush(sid)
                else:
                    ok_b = b.release(sid)
                    if ok_b:
                        a.release(sid)
                        live = [x for x in live if x[0] != sid]
                        continue
                    with pytest.raises(lz.IllegalTransition):
                        a.release(sid)
                    continue
                for x in live:
                    if x[0] == sid:
                        x[1] += 1
            assert a.live_bytes() == b.live_bytes()


def test_ring_illegal_transitions(lz):
    r = lz.RingCore(100)
    sid, _ = r.try_reserve(10, 1)
    with pytest.raises(lz.IllegalTransition):
        r.begin_flush(sid)
    with pytest.raises(lz.IllegalTransition):
        r.release(sid)
    with pytest.raises(lz.IllegalTransition):
        r.mark_filled(999)


def test_header_bytes_match_oracle(lz, oracle):
    rng = random.Random(5)
    for _ in range(300):
        n = rng.randint(0, 12)
        keys = ["".join(rng.choice("ab/_.-xyz0") for _ in range(rng.randint(0, 40))) for _ in range(n)]
        h = lz.CheckpointFileHeader([lz.HeaderEntry(k) for k in keys])
        cur = h.serialized_size()
        for e in h.entries:
            cur += rng.randint(0, 3)
            e.offset, e.length, e.checksum = cur, rng.randint(0, 1 << 40), rng.getrandbits(64)
            cur += e.length
        raw = lz.serialize_header(h)
        assert raw == oracle.header_bytes([(e.key, e.offset, e.length, e.checksum) for e in h.entries])
        assert lz.parse_header(raw) == h


def test_header_rejects_damage(lz):
    h = lz.CheckpointFileHeader([lz.HeaderEntry("k", 0, 5, 1)])
    h.entries[0].offset = h.serialized_size()
    raw = bytearray(lz.serialize_header(h))
    with pytest.raises(lz.BadMagic):
        lz.parse_header(b"NOTACKPT" + bytes(raw[8:]))
    with pytest.raises(lz.TruncatedFile):
        lz.parse_header(bytes(raw[:-3]))
    raw[20] ^= 1
    with pytest.raises(lz.FormatError):
        lz.parse_header(bytes(raw))
    bad = lz.CheckpointFileHeader([lz.HeaderEntry("k", 1, 5, 1)])  # offset inside header
    with pytest.raises(lz.FormatError):
        lz.serialize_header(bad)


def test_plan_matches_oracle(lz, oracle):
    rng = random.Random(9)
    for _ in range(200):
        dp, pp, tp = rng.randint(1, 4), rng.randint(1, 3), rng.choice([1, 2, 4])
        layers = rng.randint(pp, 50)
        params = rng.randint(1, 10 ** 9)
        bm, bo = rng.randint(1, 4), rng.randint(1, 16)
        topo = lz.ParallelTopology(dp, pp, tp, tp, dp * pp)
        plan = lz.plan_checkpoint(topo, lz.ModelSpec(param_count=params, layer_count=layers,
                                                     bytes_per_param_model=bm, bytes_per_param_optimizer=bo), 1)
        total = 0
        for r in range(topo.ranks()):
            mine = plan.shards(r)
            ref = oracle.plan_rank(dp, pp, tp, params, layers, bm, bo, r)
            assert [(s.size_bytes, s.filename) for s in mine] == [(s["size"], s["filename"]) for s in ref]
            total += sum(s.size_bytes for s in mine)
        assert total == params * (bm + bo)


def test_plan_rejects_bad_topology(lz):
    with pytest.raises(lz.ConfigError):
        lz.plan_checkpoint(lz.ParallelTopology(2, 1, 1, 4, 1), lz.ModelSpec(param_count=10, layer_count=1), 1)


def test_flatten_order_matches_oracle(lz, oracle):
    paths = ["a.b/y", "a/x", "a-b/z", "a/b/c", "A/x", "a0", "b/~", "a/b/a", "y/10", "y/2", "y/1"]
    t = lz.StateTree()
    for p in paths:
        t.set_blob(p, p.encode())
    assert [l.path for l in t.flatten()] == [paths[i] for i in oracle.flatten_order(paths)]
    with pytest.raises(lz.DuplicatePath):
        t.set_blob("a/x", b"again")
    with pytest.raises(lz.DuplicatePath):
        t.set_blob("a/x/deeper", b"through a leaf")
    assert t.blob_at("a0") == b"a0"


def test_manifest_roundtrip_and_errors(lz, tmp_path):
    m = lz.ManifestStore(tmp_path / "manifest.json")
    assert m.latest_committed() is None
    m.commit_step(3, [("step-3/rank-0-0-0/a.ckpt", 10, 0xABC)])
    m.commit_step(1, [("step-1/rank-0-0-0/a.ckpt", 5, 1)])
    again = lz.ManifestStore(tmp_path / "manifest.json")
    assert again.latest_committed() == 3 and again.is_committed(1) and not again.is_committed(2)
    text = (tmp_path / "manifest.json").read_text()
    assert '"digest": "0000000000000abc"' in text and '"format": "lzckpt-manifest-1"' in text
    (tmp_path / "bad.json").write_text("{not json")
    with pytest.raises(lz.CorruptManifest):
        lz.ManifestStore(tmp_path / "bad.json")


def test_device_calls_fail_loudly_without_gpu(lz):
    if lz.device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(lz.DeviceError):
        lz.DeviceRegion(64)


CPU_SUITES = ["test_ring", "test_format", "test_topology", "test_manifest"]


@pytest.mark.parametrize("suite", CPU_SUITES)
def test_reference_suite_on_cpu(suite):
    """The reference's own doctest sources (compiled in place against our
    headers + library by tests/reftests/Makefile) for the host-only modules."""
    exe = os.path.join(ROOT, "tests", "reftests", "bin", suite)
    if not os.path.exists(exe):
        pytest.skip("reference suites not built (needs /root/reference at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    assert " 0 failed" in r.stderr.splitlines()[-1]
