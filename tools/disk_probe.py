"""Local-disk write throughput: buffered+fsync vs O_DIRECT with N writer
threads (8 GiB, 64 MiB pieces).  python tools/disk_probe.py"""
import mmap
import os
import threading
import time

PATH = "/tmp/lzk_disk_probe"
TOTAL, PIECE = 8 << 30, 64 << 20


def run(threads, direct):
    flags = os.O_WRONLY | os.O_CREAT | os.O_TRUNC | (os.O_DIRECT if direct else 0)
    fd = os.open(PATH, flags, 0o644)
    bufs = [mmap.mmap(-1, PIECE) for _ in range(threads)]  # page-aligned
    for b in bufs:
        b.write(os.urandom(1 << 20) * (PIECE >> 20))
    offs = list(range(0, TOTAL, PIECE))
    lock = threading.Lock()

    def worker(k):
        while True:
            with lock:
                if not offs:
                    return
                o = offs.pop()
            os.pwrite(fd, bufs[k], o)
    t0 = time.perf_counter()
    th = [threading.Thread(target=worker, args=(k,)) for k in range(threads)]
    [t.start() for t in th]
    [t.join() for t in th]
    os.fsync(fd)
    dt = time.perf_counter() - t0
    os.close(fd)
    os.unlink(PATH)
    return TOTAL / dt / 1e9


for direct in (False, True):
    for th in (1, 4, 8, 16):
        print(f"{'O_DIRECT' if direct else 'buffered'} threads={th}: {run(th, direct):.2f} GB/s", flush=True)
