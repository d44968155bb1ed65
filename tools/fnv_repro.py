"""Debug helper for lzk_fnv1a64_batch: python tools/fnv_repro.py <case>."""
import ctypes as C
import subprocess
import sys

import numpy as np

sys.path.insert(0, '/root/repo')
import paper_2406_10707_b200 as lz  # noqa: E402
from paper_2406_10707_b200 import _native as N  # noqa: E402


def run(case):
    from oracle import oracle as O
    n = 1 << 20
    host = np.random.default_rng(1).integers(0, 256, n, dtype=np.uint8)
    p = C.c_void_p()
    assert lz.dev.lzk_dev_alloc(0, n, C.byref(p)) == 0
    assert lz.dev.lzk_memcpy_h2d(0, p.value, host.ctypes.data, n) == 0
    s = C.c_void_p()
    assert lz.dev.lzk_stream_create(0, 0, C.byref(s)) == 0
    mode, L, ctas = case.split(":")
    L, ctas = int(L), int(ctas)
    if mode == "dev":
        o = C.c_void_p()
        assert lz.dev.lzk_dev_alloc(0, 64, C.byref(o)) == 0
    else:
        o = C.c_void_p()
        assert lz.dev.lzk_host_alloc(64, 1, C.byref(o)) == 0
    arr = (N.HashDescC * 1)(N.HashDescC(p.value, L, lz.FNV_BASIS, o.value))
    rc = lz.dev.lzk_fnv1a64_batch(s, arr, 1, ctas)
    rc2 = lz.dev.lzk_stream_sync(s)
    got = np.zeros(1, dtype=np.uint64)
    if rc2 == 0:
        if mode == "dev":
            lz.dev.lzk_memcpy_d2h(0, got.ctypes.data, o.value, 8)
        else:
            got[0] = C.c_uint64.from_address(o.value).value
    print(case, rc, rc2, lz.dev.lzk_last_error().decode(), rc2 == 0 and int(got[0]) == O.fnv64(host[:L]), flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1:
        run(sys.argv[1])
    else:
        for case in ["dev:0:1", "map:0:1", "dev:0:0", "dev:5000:1", "dev:100000:0", "map:100000:3"]:
            subprocess.run([sys.executable, __file__, case])
