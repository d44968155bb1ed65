"""Where restore time goes: write a C2 slice checkpoint, then time
(a) raw parallel pread of its files (page cache warm, then cold after
drop_caches when permitted), (b) Engine.restore with device checksums.
    python tools/restore_probe.py [layers]"""
import ctypes as C
import json
import os
import shutil
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_10707_b200 as lz  # noqa: E402
from paper_2406_10707_b200.workloads import llama7b_shard  # noqa: E402

layers = int(sys.argv[1]) if len(sys.argv) > 1 else 2
tmp = "/tmp/rprobe"
shutil.rmtree(tmp, ignore_errors=True)
os.makedirs(tmp)
w = llama7b_shard(layers=layers, vocab=8000, name="probe")
built = lz.build_workload(w.write_spec(os.path.join(tmp, "p.spec")), 0)
cfg = lz.EngineConfig(checkpoint_root=tmp + "/ck", host_buffer_bytes=int(built.bytes * 1.01) + (64 << 20),
                      fsync_on_finalize=True)
eng = lz.Engine(cfg, built.topo, built.rank)
plan = lz.plan_checkpoint(built.topo, built.model, built.step)
t = eng.capture(plan, built.tree, 9)
eng.update_barrier(t)
eng.wait_persisted(t)
files = [os.path.join(tmp, "ck", f) for f in t.shard_files()]
m = lz.ManifestStore(tmp + "/ck/manifest.json")
m.commit_step(9, lz.committed_record(t, tmp + "/ck"))
total = sum(os.path.getsize(f) for f in files)
out = {"bytes": total}


def pread_all(threads, piece=64 << 20):
    buf = bytearray(piece * threads)
    mv = memoryview(buf)
    jobs = [(f, o) for f in files for o in range(0, os.path.getsize(f), piece)]
    lock = threading.Lock()

    def worker(k):
        fds = {}
        while True:
            with lock:
                if not jobs:
                    break
                f, o = jobs.pop()
            fd = fds.setdefault(f, os.open(f, os.O_RDONLY))
            os.preadv(fd, [mv[k * piece:(k + 1) * piece]], o)
        for fd in fds.values():
            os.close(fd)
    t0 = time.perf_counter()
    th = [threading.Thread(target=worker, args=(k,)) for k in range(threads)]
    [x.start() for x in th]
    [x.join() for x in th]
    return total / (time.perf_counter() - t0) / 1e9


for th in (1, 8, 16):
    out[f"pread_warm_{th}t_gbps"] = round(pread_all(th), 3)
t0 = time.perf_counter()
back = eng.restore(m, 9)
out["restore_warm_gbps"] = round(total / (time.perf_counter() - t0) / 1e9, 3)
del back
try:
    os.sync()
    with open("/proc/sys/vm/drop_caches", "w") as f:
        f.write("3\n")
    out["pread_cold_8t_gbps"] = round(pread_all(8), 3)
    with open("/proc/sys/vm/drop_caches", "w") as f:
        f.write("3\n")
    t0 = time.perf_counter()
    back = eng.restore(m, 9)
    out["restore_cold_gbps"] = round(total / (time.perf_counter() - t0) / 1e9, 3)
    del back
except OSError as e:
    out["drop_caches"] = str(e)
eng.close()
shutil.rmtree(tmp, ignore_errors=True)
print(json.dumps(out))
