"""Why the engine's copy-engine path can trail the box's 8 GiB DMA probe.
Same box, same pinned-memory kind (mmap + THP + cudaHostRegister), D2H GB/s:
  A  probe: 8 GiB device buffer -> 8 GiB host buffer, 256 MiB DMAs
  B  one source buffer -> a host buffer of the C2 shard size (107.8 GB),
     256 MiB DMAs sweeping the whole range
  C  the 1164 C2 tensors -> that big buffer, one DMA per tensor (piecewise
     <= 256 MiB), in engine order
  D  the engine itself (copy-engine variant, host-memory tier)
Prints one JSON line.  python tools/dma_gap.py"""
import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_10707_b200 as lz  # noqa: E402
from paper_2406_10707_b200 import _native as N  # noqa: E402
from paper_2406_10707_b200.workloads import llama7b_shard  # noqa: E402

d = lz.dev


def ck(rc):
    if rc:
        raise RuntimeError(d.lzk_last_error().decode())


s = C.c_void_p()
ck(d.lzk_stream_create(0, 0, C.byref(s)))
e0, e1 = C.c_void_p(), C.c_void_p()
ck(d.lzk_event_create(0, 0, C.byref(e0)))
ck(d.lzk_event_create(0, 0, C.byref(e1)))


slow_prio = C.c_void_p()
ck(d.lzk_stream_create(0, 1, C.byref(slow_prio)))
gev = C.c_void_p()
ck(d.lzk_event_create(0, 0, C.byref(gev)))


def timed(descs, reps=2, stream=None, group=0):
    st = stream or s
    arr = (N.CopyDescC * len(descs))(*[N.CopyDescC(*x) for x in descs])
    total = sum(x[2] for x in descs)
    best = 0.0
    for _ in range(reps):
        ck(d.lzk_event_record(e0, st))
        if group:
            i, acc, start = 0, 0, 0
            while i < len(descs):
                acc += descs[i][2]
                i += 1
                if acc >= group or i == len(descs):
                    sub = C.cast(C.byref(arr, start * C.sizeof(N.CopyDescC)), C.POINTER(N.CopyDescC))
                    ck(d.lzk_ce_copy_d2h(st, sub, i - start))
                    ck(d.lzk_event_record(gev, st))
                    start, acc = i, 0
        else:
            ck(d.lzk_ce_copy_d2h(st, arr, len(descs)))
        ck(d.lzk_event_record(e1, st))
        ck(d.lzk_stream_sync(st))
        ms = C.c_float()
        ck(d.lzk_event_elapsed_ms(e0, e1, C.byref(ms)))
        best = max(best, total / (ms.value * 1e-3) / 1e9)
    return round(best, 2)


out = {}
w = llama7b_shard()
built = lz.build_workload(w.write_spec("/tmp/dma_gap.spec"), 0)
big = built.bytes
src8 = C.c_void_p()
ck(d.lzk_dev_alloc(0, 8 << 30, C.byref(src8)))
host = C.c_void_p()
t0 = time.time()
ck(d.lzk_host_alloc(big, 1 | 2, C.byref(host)))
out["pin_s"] = round(time.time() - t0, 2)
chunk = 256 << 20
# A: probe shape on the first 8 GiB of the big buffer
out["A_probe_8GiB"] = timed([(src8.value + o, host.value + o, chunk) for o in range(0, 8 << 30, chunk)], 3)
# B: sweep the whole big range from one 8 GiB source
out["B_sweep_108GB"] = timed([(src8.value + (o % (8 << 30)), host.value + o, min(chunk, big - o))
                              for o in range(0, big, chunk)])
# C: the C2 tensors, engine order (flatten order of the tree), per tensor, <= 256 MiB pieces
leaves = [l for l in built.tree.flatten() if l.is_region]
descs, off = [], 0
for l in leaves:
    r = built.tree.region_at(l.path)
    for p in range(0, l.size, chunk):
        n = min(chunk, l.size - p)
        descs.append((r.device_ptr + p, host.value + off + p, n))
    off += l.size
out["C_tensors_108GB"] = timed(descs)
for mis in (6, 14, 64, 128, 256, 2048):
    out[f"C_dst_plus_{mis}"] = timed([(a, b + mis, n) for a, b, n in descs if b + mis + n <= host.value + big])
out["C_low_priority_stream"] = timed(descs, stream=slow_prio)
out["C_event_per_256MB"] = timed(descs, group=256 << 20)
d.lzk_host_free(host)
# D: the engine itself
cfg = lz.EngineConfig(checkpoint_root="/tmp/dma_gap_ck", host_buffer_bytes=int(big * 1.01) + (256 << 20),
                      large_leaf_threshold=1 << 20, fsync_on_finalize=False, flush_discard=True, hugepages=True)
eng = lz.Engine(cfg, built.topo, built.rank)
plan = lz.plan_checkpoint(built.topo, built.model, built.step)
eng.set_copy_variant(force_copy_engine=True)
best = 0.0
for st in range(3):
    t = eng.capture(plan, built.tree, st + 1)
    eng.update_barrier(t)
    eng.wait_persisted(t)
    if st:
        best = max(best, t.payload_bytes() / (eng.ticket_device_ms(t) * 1e-3) / 1e9)
out["D_engine_ce"] = round(best, 2)
eng.set_copy_variant(force_copy_engine=True, group_bytes=8 << 30)
best = 0.0
for st in range(3):
    t = eng.capture(plan, built.tree, 10 + st)
    eng.update_barrier(t)
    eng.wait_persisted(t)
    if st:
        best = max(best, t.payload_bytes() / (eng.ticket_device_ms(t) * 1e-3) / 1e9)
out["D_engine_ce_groups_8GiB"] = round(best, 2)
eng.close()
print(json.dumps(out))
