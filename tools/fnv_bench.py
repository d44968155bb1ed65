"""Throughput of the device FNV-1a-64 kernel (lzk_fnv1a64_batch).

    python tools/fnv_bench.py

Cases (device-resident inputs, a 4 GiB buffer > L2, timed with CUDA events
on the launching stream, best of 3):
  * c2      — the 1164 C2 (LLaMA-7B shard) entry sizes, 107.8 GB total,
              mapped cyclically onto the buffer; swept over grid sizes
  * uniform — 4096 x 1 MiB entries
  * single  — one 1 GiB entry: at 1 CTA one warp's chain (the per-warp
              rate), with more CTAs the segmented multi-pass schedule
  * window  — a 512 MiB restore window holding two entry slices
One JSON line per (case, ctas).
"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_10707_b200 as lz  # noqa: E402
from paper_2406_10707_b200 import _native as N  # noqa: E402
from paper_2406_10707_b200.workloads import llama7b_shard  # noqa: E402

d = lz.dev


def ck(rc):
    if rc:
        raise RuntimeError(d.lzk_last_error().decode())


BUF = 4 << 30
p = C.c_void_p()
ck(d.lzk_dev_alloc(0, BUF, C.byref(p)))
s = C.c_void_p()
ck(d.lzk_stream_create(0, 0, C.byref(s)))
ck(d.lzk_fill_splitmix(s, p.value, BUF, 5, 0))
out = C.c_void_p()
ck(d.lzk_dev_alloc(0, 8 << 16, C.byref(out)))
e0, e1 = C.c_void_p(), C.c_void_p()
ck(d.lzk_event_create(0, 0, C.byref(e0)))
ck(d.lzk_event_create(0, 0, C.byref(e1)))


def descs(sizes):
    arr = (N.HashDescC * len(sizes))()
    off = 0
    for i, n in enumerate(sizes):
        if off + n > BUF:
            off = 0
        arr[i] = N.HashDescC(p.value + off, n, lz.FNV_BASIS, out.value + 8 * i)
        off += (n + 255) // 256 * 256
    return arr


def run(name, sizes, ctas_list):
    arr = descs(sizes)
    total = sum(sizes)
    for ctas in ctas_list:
        best = None
        for _ in range(3):
            ck(d.lzk_event_record(e0, s))
            ck(d.lzk_fnv1a64_batch(s, arr, len(sizes), ctas))
            ck(d.lzk_event_record(e1, s))
            ck(d.lzk_stream_sync(s))
            ms = C.c_float()
            ck(d.lzk_event_elapsed_ms(e0, e1, C.byref(ms)))
            best = ms.value if best is None else min(best, ms.value)
        print(json.dumps({"case": name, "entries": len(sizes), "bytes": total, "ctas": ctas,
                          "ms": round(best, 3), "GBps": round(total / best / 1e6, 2),
                          "GBps_per_cta": round(total / best / 1e6 / (ctas or 1), 2) if ctas else None}),
              flush=True)


if not os.environ.get("FNV_BENCH_ONLY_CONT"):
    c2 = [sz for kind, _, sz in llama7b_shard().leaves if kind == "r"]
    run("c2", c2, [1, 2, 4, 8, 16, 32, 64, 148, 0])
    run("uniform", [1 << 20] * 4096, [1, 8, 16, 148, 0])
    run("single", [1 << 30], [1, 16, 148, 0])
    run("window", [300 << 20, 212 << 20], [16, 148, 0])


def run_cont(name, sizes, mapped, cont, ctas=0, odd=True):
    """Restore-like call: slices at odd offsets, states in mapped host or
    device memory, continue mode."""
    st = C.c_void_p()
    if mapped:
        ck(d.lzk_host_alloc(8 * len(sizes), 1, C.byref(st)))
    else:
        ck(d.lzk_dev_alloc(0, 8 * len(sizes), C.byref(st)))
    arr = (N.HashDescC * len(sizes))()
    off = 5 if odd else 0
    for i, n in enumerate(sizes):
        arr[i] = N.HashDescC(p.value + off, n, lz.FNV_BASIS, st.value + 8 * i)
        off += n
    fn = d.lzk_fnv1a64_continue if cont else d.lzk_fnv1a64_batch
    best = None
    for _ in range(3):
        ck(d.lzk_event_record(e0, s))
        ck(fn(s, arr, len(sizes), ctas))
        ck(d.lzk_event_record(e1, s))
        ck(d.lzk_stream_sync(s))
        ms = C.c_float()
        ck(d.lzk_event_elapsed_ms(e0, e1, C.byref(ms)))
        best = ms.value if best is None else min(best, ms.value)
    print(json.dumps({"case": name, "mapped_out": mapped, "continue": cont, "odd": odd, "entries": len(sizes),
                      "bytes": sum(sizes), "ms": round(best, 3), "GBps": round(sum(sizes) / best / 1e6, 2)}),
          flush=True)


if os.environ.get("FNV_BENCH_ONLY_CONT"):
    sl = [67108864 - 1000, 67108864, 67108864 + 3, 67108864, 67108864, 67108864, 67108864, 67108864 - 7000]
    for mapped in (False, True):
        for cont in (False, True):
            run_cont("restore_window", sl, mapped, cont)
    run_cont("restore_window", sl, True, True, odd=False)
