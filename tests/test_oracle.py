"""Pins the oracle (oracle/lzk_oracle.c) before it is trusted as the checker:
FNV-1a known answers, the reference's golden C1 digests, and
fixtures produced by running the reference engine itself
(tests/golden/ref_fixtures.json from tests/golden/make_fixtures.py)."""
import pytest

FNV_KAT = {b"": 0xCBF29CE484222325, b"a": 0xAF63DC4C8601EC8C, b"foobar": 0x85944171F73967E8}
C1_GOLDEN = {"step-1/rank-0-0-0/layers-0-11.ckpt": (248887594, 0x18D06AB61AFAE34A),
             "step-1/rank-0-0-0/optimizer-0.ckpt": (1493305660, 0xC1F7BF0708955268)}


def test_fnv_known_answers(oracle):
    for data, want in FNV_KAT.items():
        assert oracle.fnv64(data) == want


def test_oracle_reproduces_reference_fixtures(oracle, cases, fixtures):
    assert set(cases) == set(fixtures)
    for name, (w, thr) in cases.items():
        files = oracle.compose_files(w, thr)
        want = fixtures[name]["files"]
        assert set(files) == set(want), name
        for rel, buf in files.items():
            assert buf.size == want[rel]["size"], (name, rel)
            assert f"{oracle.fnv64(buf):016x}" == want[rel]["fnv"], (name, rel)


def test_oracle_reproduces_golden_c1_digests(oracle):
    from paper_2406_10707_b200.workloads import gpt2_small
    files = oracle.compose_files(gpt2_small(), 1 << 20)
    assert {k: (v.size, oracle.fnv64(v)) for k, v in files.items()} == C1_GOLDEN


def test_oracle_flatten_order_is_per_component(oracle):
    paths = ["a.b/y", "a/x", "a-b/z", "a/b/c", "A/x", "a0", "b/~", "a/b/a"]
    order = [paths[i] for i in oracle.flatten_order(paths)]
    # std::map per component: "a" < "a-b" < "a.b" < "a0" bytewise, and a/... before a-b/...
    assert order == ["A/x", "a/b/a", "a/b/c", "a/x", "a-b/z", "a.b/y", "a0", "b/~"]


def test_oracle_ring_wraps_with_gap(oracle):
    r = oracle.Ring(100)
    a = r.try_reserve(40)
    b = r.try_reserve(40)
    assert a == (1, 0) and b == (2, 40)
    assert r.try_reserve(30) is None  # 20 left at the tail, 0 at the head
    for sid in (1,):
        assert r.mark_filled(sid) and r.begin_flush(sid) and r.release(sid)
    c = r.try_reserve(30)  # tail run of 20 too short: wraps to 0, leaves a gap
    assert c == (3, 0)
    assert not r.release(3)  # FIFO: segment 2 is older
