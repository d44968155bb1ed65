"""Local-disk throughput: writes (buffered+fsync vs O_DIRECT) and O_DIRECT
reads, with N threads (8 GiB, 64 MiB pieces).
    python tools/disk_probe.py [write|read|all]"""
import mmap
import os
import sys
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


def run_read(threads, piece):
    """O_DIRECT reads of an 8 GiB file written just before (not cached)."""
    fd = os.open(PATH, os.O_WRONLY | os.O_CREAT | os.O_TRUNC | os.O_DIRECT, 0o644)
    buf = mmap.mmap(-1, PIECE)
    buf.write(os.urandom(1 << 20) * (PIECE >> 20))
    for o in range(0, TOTAL, PIECE):
        os.pwrite(fd, buf, o)
    os.fsync(fd)
    os.close(fd)
    fd = os.open(PATH, os.O_RDONLY | os.O_DIRECT)
    bufs = [mmap.mmap(-1, piece) for _ in range(threads)]
    offs = list(range(0, TOTAL, piece))
    lock = threading.Lock()

    def worker(k):
        while True:
            with lock:
                if not offs:
                    return
                o = offs.pop(0)
            os.preadv(fd, [bufs[k]], o)
    t0 = time.perf_counter()
    th = [threading.Thread(target=worker, args=(k,)) for k in range(threads)]
    [t.start() for t in th]
    [t.join() for t in th]
    dt = time.perf_counter() - t0
    os.close(fd)
    os.unlink(PATH)
    return TOTAL / dt / 1e9


mode = sys.argv[1] if len(sys.argv) > 1 else "write"
if mode in ("write", "all"):
    for direct in (False, True):
        for th in (1, 4, 8, 16):
            print(f"{'O_DIRECT' if direct else 'buffered'} threads={th}: {run(th, direct):.2f} GB/s", flush=True)
if mode in ("read", "all"):
    for piece in (16 << 20, 64 << 20):
        for th in (1, 2, 4, 8):
            print(f"O_DIRECT read piece={piece >> 20}MiB threads={th}: {run_read(th, piece):.2f} GB/s", flush=True)
