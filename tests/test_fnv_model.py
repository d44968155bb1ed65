"""CPU check of the device FNV-1a-64 schedules (lzk_fnv.cu) through their
executable model (tools/fnv_scan_model.py): the bit-sliced warp scan, the
single-plane multi-pass schedule and the dual-plane passes + resolve used for
long ranges all reproduce the byte-serial reference fold
(include/lzckpt/checksum.hpp; reference checksum.hpp:17-24)."""
import os
import random
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
import fnv_scan_model as M  # noqa: E402


def test_warp_scan_model_matches_fnv():
    rng = random.Random(3)
    for n in (0, 1, 1023, 1024, 2049):
        d = bytes(rng.getrandbits(8) for _ in range(n))
        h0 = rng.getrandbits(64)
        assert M.fnv_model(d, h0) == M.fnv(d, h0)


def test_dual_plane_schedule_matches_fnv():
    rng = random.Random(5)
    for n, seglen in ((4 * 1024 + 13, 1024), (6 * 1024, 2048)):
        d = bytes(rng.getrandbits(8) for _ in range(n))
        h0 = rng.getrandbits(64)
        assert M.segmented_dual(d, h0, seglen) == M.fnv(d, h0)
