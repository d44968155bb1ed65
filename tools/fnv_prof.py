"""One lzk_fnv_kernel launch per grid size over 4096 x 1 MiB device ranges
(ncu target): python tools/fnv_prof.py 8 148"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_10707_b200 as lz  # noqa: E402
from paper_2406_10707_b200 import _native as N  # noqa: E402

d = lz.dev
BUF = 4 << 30
p, s, out = C.c_void_p(), C.c_void_p(), C.c_void_p()
assert d.lzk_dev_alloc(0, BUF, C.byref(p)) == 0
assert d.lzk_stream_create(0, 0, C.byref(s)) == 0
assert d.lzk_fill_splitmix(s, p.value, BUF, 5, 0) == 0
assert d.lzk_dev_alloc(0, 8 * 4096, C.byref(out)) == 0
arr = (N.HashDescC * 4096)(*[N.HashDescC(p.value + (i << 20), 1 << 20, lz.FNV_BASIS, out.value + 8 * i)
                             for i in range(4096)])
for ctas in [int(x) for x in sys.argv[1:]]:
    assert d.lzk_fnv1a64_batch(s, arr, 4096, ctas) == 0
    assert d.lzk_stream_sync(s) == 0
print("ok")
