"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes front-end of oracle/liboracle.so (the plain-C restatement of the
reference's snapshot-path algorithms, oracle/lzk_oracle.c). Only tests/,
__graft_entry__.smoke() and bench.py's CPU-baseline leg import this module,
and only as the checker: it composes the exact shard files the reference
writes for a workload, so the product's files can be compared byte for byte.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Dict, List, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "liboracle.so")
REF_DRIVER = os.path.join(HERE, "_ref", "ref_snapshot")
FNV_BASIS = 0xCBF29CE484222325


def build() -> str:
    """Compile the C restatement (gcc, seconds)."""
    subprocess.run(["make", "-C", HERE, "oracle"], check=True, capture_output=True)
    return SO


def _load():
    if not os.path.exists(SO):
        build()
    lib = C.CDLL(SO)
    u8p, u64, u32 = C.c_void_p, C.c_uint64, C.c_uint32
    lib.lzo_fnv1a64.restype = u64
    lib.lzo_fnv1a64.argtypes = [u64, u8p, u64]
    lib.lzo_fill_mt19937_64.argtypes = [u64, u64, C.POINTER(u64), C.POINTER(C.c_void_p)]
    lib.lzo_fill_splitmix.argtypes = [u64, u64, u64, u8p]
    lib.lzo_splitmix_fnv.restype = u64
    lib.lzo_splitmix_fnv.argtypes = [u64, u64, u64]
    lib.lzo_ring_new.restype = C.c_void_p
    lib.lzo_ring_new.argtypes = [u64]
    lib.lzo_ring_free.argtypes = [C.c_void_p]
    lib.lzo_ring_try_reserve.argtypes = [C.c_void_p, u64, C.POINTER(u64), C.POINTER(u64)]
    for f in ("lzo_ring_mark_filled", "lzo_ring_begin_flush", "lzo_ring_release"):
        getattr(lib, f).argtypes = [C.c_void_p, u64]
    lib.lzo_ring_live_bytes.restype = u64
    lib.lzo_ring_live_bytes.argtypes = [C.c_void_p]
    lib.lzo_header_size.restype = u64
    lib.lzo_header_size.argtypes = [u32, C.POINTER(u32)]
    lib.lzo_header_serialize.restype = u64
    lib.lzo_header_serialize.argtypes = [u32, C.POINTER(C.c_char_p), C.POINTER(u32), C.POINTER(u64),
                                         C.POINTER(u64), C.POINTER(u64), u8p]
    lib.lzo_flatten_order.argtypes = [u32, C.POINTER(C.c_char_p), C.POINTER(u32)]
    lib.lzo_compose_shard.restype = u64
    lib.lzo_compose_shard.argtypes = [u32, C.POINTER(C.c_char_p), C.POINTER(C.c_uint8), C.POINTER(u64),
                                      C.POINTER(C.c_void_p), u64, u8p]
    lib.lzo_plan_rank.restype = C.c_int
    lib.lzo_plan_rank.argtypes = [u32, u32, u32, u64, u32, u32, u32, u32] + [C.POINTER(u32), C.POINTER(u64),
                                                                            C.POINTER(u32), C.POINTER(u32),
                                                                            C.POINTER(u32)]
    return lib


L = _load()


def fnv64(data, state: int = FNV_BASIS) -> int:
    a = np.frombuffer(data, dtype=np.uint8) if not isinstance(data, np.ndarray) else data
    return L.lzo_fnv1a64(state, a.ctypes.data if a.size else None, a.size)


def plan_rank(dp, pp, tp, params, layers, bpp_model, bpp_opt, flat_rank) -> List[dict]:
    kind = (C.c_uint32 * 2)()
    size = (C.c_uint64 * 2)()
    first = (C.c_uint32 * 2)()
    cnt = (C.c_uint32 * 2)()
    part = (C.c_uint32 * 2)()
    n = L.lzo_plan_rank(dp, pp, tp, params, layers, bpp_model, bpp_opt, flat_rank, kind, size, first, cnt, part)
    out = []
    for i in range(n):
        if kind[i] == 0:
            fname = f"layers-{first[i]}-{first[i] + (cnt[i] - 1 if cnt[i] else 0)}.ckpt"
        else:
            fname = f"optimizer-{part[i]}.ckpt"
        out.append(dict(kind=kind[i], size=size[i], first_layer=first[i], layer_count=cnt[i],
                        partition=part[i], filename=fname))
    return out


def flatten_order(paths: List[str]) -> List[int]:
    n = len(paths)
    arr = (C.c_char_p * n)(*[p.encode() for p in paths])
    order = (C.c_uint32 * n)()
    L.lzo_flatten_order(n, arr, order)
    return list(order)


def generate(workload) -> List[np.ndarray]:
    """Leaf bytes in spec (fill) order, with the workload's generator."""
    sizes = [s for _, _, s in workload.leaves]
    bufs = [np.empty(max(s, 1), dtype=np.uint8) for s in sizes]
    if workload.gen == "mt19937_64":
        n = len(sizes)
        L.lzo_fill_mt19937_64(workload.seed, n, (C.c_uint64 * n)(*sizes),
                              (C.c_void_p * n)(*[b.ctypes.data for b in bufs]))
    else:
        for i, (b, s) in enumerate(zip(bufs, sizes)):
            L.lzo_fill_splitmix(workload.seed, i, s, b.ctypes.data)
    return [b[:s] for b, s in zip(bufs, sizes)]


def compose_files(workload, threshold: int, data: List[np.ndarray] = None) -> Dict[str, np.ndarray]:
    """{relative shard path: file bytes} the reference engine writes for one
    capture of `workload` at its step (engine.cpp:96-231 flow)."""
    if data is None:
        data = generate(workload)
    dp, pp, tp, gpn, nodes = workload.topology
    rdp, rpp, rtp = workload.rank
    flat = (rdp * pp + rpp) * tp + rtp
    shards = plan_rank(dp, pp, tp, workload.param_count, workload.layer_count, workload.bpp_model,
                       workload.bpp_opt, flat)
    tops = sorted({p.split("/")[0] for _, p, _ in workload.leaves}, key=lambda s: s.encode())
    if len(tops) != len(shards):
        raise ValueError(f"{len(tops)} top-level children vs {len(shards)} shards")
    out = {}
    for top, sh in zip(tops, shards):
        idx = [i for i, (_, p, _) in enumerate(workload.leaves) if p.split("/")[0] == top]
        paths = [workload.leaves[i][1] for i in idx]
        order = [idx[j] for j in flatten_order(paths)]
        total = sum(workload.leaves[i][2] for i in order)
        if total != sh["size"]:
            raise ValueError(f"subtree {top}: {total} bytes vs shard {sh['size']}")
        n = len(order)
        cpaths = (C.c_char_p * n)(*[workload.leaves[i][1].encode() for i in order])
        isr = (C.c_uint8 * n)(*[1 if workload.leaves[i][0] == "r" else 0 for i in order])
        sizes = (C.c_uint64 * n)(*[workload.leaves[i][2] for i in order])
        ptrs = (C.c_void_p * n)(*[data[i].ctypes.data if data[i].size else None for i in order])
        fsize = L.lzo_compose_shard(n, cpaths, isr, sizes, ptrs, threshold, None)
        buf = np.empty(fsize, dtype=np.uint8)
        L.lzo_compose_shard(n, cpaths, isr, sizes, ptrs, threshold, buf.ctypes.data)
        rel = f"step-{workload.step}/rank-{rdp}-{rpp}-{rtp}/{sh['filename']}"
        out[rel] = buf
    return out


class Ring:
    """Oracle ring (ring_core.cpp:21-139)."""

    def __init__(self, cap):
        self.h = L.lzo_ring_new(cap)

    def __del__(self):
        if getattr(self, "h", None):
            L.lzo_ring_free(self.h)
            self.h = None

    def try_reserve(self, size):
        i, o = C.c_uint64(), C.c_uint64()
        return (i.value, o.value) if L.lzo_ring_try_reserve(self.h, size, C.byref(i), C.byref(o)) else None

    def mark_filled(self, i):
        return L.lzo_ring_mark_filled(self.h, i) == 0

    def begin_flush(self, i):
        return L.lzo_ring_begin_flush(self.h, i) == 0

    def release(self, i):
        return L.lzo_ring_release(self.h, i) == 0

    def live_bytes(self):
        return L.lzo_ring_live_bytes(self.h)


def header_bytes(entries: List[Tuple[str, int, int, int]]) -> bytes:
    n = len(entries)
    keys = [e[0].encode() for e in entries]
    klen = (C.c_uint32 * n)(*[len(k) for k in keys])
    size = L.lzo_header_size(n, klen)
    buf = np.empty(size, dtype=np.uint8)
    L.lzo_header_serialize(n, (C.c_char_p * n)(*keys), klen, (C.c_uint64 * n)(*[e[1] for e in entries]),
                           (C.c_uint64 * n)(*[e[2] for e in entries]), (C.c_uint64 * n)(*[e[3] for e in entries]),
                           buf.ctypes.data)
    return buf.tobytes()


def expected_headers(workload, threshold: int, threads: int = 16):
    """Headers (key, offset, length, checksum) of every shard file of a
    splitmix64 workload, computed WITHOUT materializing the payload: large
    leaves hash their generated stream in C (threads release the GIL), the
    __meta__ entry is composed from the (small) inline leaves. For GB-scale
    full-size parity: compare with the engine's finalized headers."""
    import struct
    from concurrent.futures import ThreadPoolExecutor
    assert workload.gen == "splitmix64"
    dp, pp, tp, gpn, nodes = workload.topology
    rdp, rpp, rtp = workload.rank
    flat = (rdp * pp + rpp) * tp + rtp
    shards = plan_rank(dp, pp, tp, workload.param_count, workload.layer_count, workload.bpp_model,
                       workload.bpp_opt, flat)
    tops = sorted({p.split("/")[0] for _, p, _ in workload.leaves}, key=lambda s: s.encode())
    big = [(i, s) for i, (_, _, s) in enumerate(workload.leaves) if s >= threshold]
    big.sort(key=lambda x: -x[1])
    with ThreadPoolExecutor(threads) as ex:
        digests = dict(zip([i for i, _ in big],
                           ex.map(lambda x: L.lzo_splitmix_fnv(workload.seed, x[0], x[1]), big)))
    out = {}
    for top, sh in zip(tops, shards):
        idx = [i for i, (_, p, _) in enumerate(workload.leaves) if p.split("/")[0] == top]
        order = [idx[j] for j in flatten_order([workload.leaves[i][1] for i in idx])]
        meta = [struct.pack("<I", len(order))]
        large = []
        for i in order:
            kind, path, size = workload.leaves[i]
            pb = path.encode()
            inl = size < threshold
            meta.append(struct.pack("<I", len(pb)) + pb + struct.pack("<BQ", (1 if kind == "r" else 0) | (2 if inl else 0), size))
            if inl:
                b = np.empty(max(size, 1), dtype=np.uint8)
                L.lzo_fill_splitmix(workload.seed, i, size, b.ctypes.data)
                meta.append(b[:size].tobytes())
            else:
                large.append((path, size, digests[i]))
        mb = b"".join(meta)
        entries = [("__meta__", len(mb), fnv64(mb))] + large
        cur = 24 + sum(28 + len(k.encode()) for k, _, _ in entries)
        hdr = []
        for k, n, d in entries:
            hdr.append((k, cur, n, d))
            cur += n
        out[f"step-{workload.step}/rank-{rdp}-{rpp}-{rtp}/{sh['filename']}"] = hdr
    return out
