"""Cold restore read settings on the GPU box's disk: writes and commits one
durable C2 sample (the e2e workload), then restores it in child processes
per (LZCKPT_READ_THREADS, LZCKPT_READ_PIECE_MB), interleaved over rounds.
The files were written with O_DIRECT and are read with O_DIRECT, so every
restore reads the disk. Prints the median GB/s per setting.

    python tools/restore_read_probe.py [layers] [rounds] [pause_s]
"""
import json
import os
import shutil
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SETTINGS = [(8, 64), (1, 16), (2, 16), (4, 16), (1, 32), (2, 32), (2, 64)]

CHILD = r"""
import os, sys, time
sys.path.insert(0, os.environ["LZK_ROOT"])
import paper_2406_10707_b200 as lz
tmp = os.environ["LZK_TMP"]
eng = lz.Engine(lz.EngineConfig(checkpoint_root=os.path.join(tmp, "ckpt"), host_buffer_bytes=64 << 20, device=0),
                lz.ParallelTopology(1, 1, 1, 1, 1), lz.RankCoord())
m = lz.ManifestStore(os.path.join(tmp, "manifest.json"))
t0 = time.perf_counter()
back = eng.restore(m, 1)
dt = time.perf_counter() - t0
print("GBPS", int(os.environ["LZK_BYTES"]) / dt / 1e9)
"""


def main():
    layers = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    pause = float(sys.argv[3]) if len(sys.argv) > 3 else 5.0
    sys.path.insert(0, ROOT)
    import paper_2406_10707_b200 as lz
    from paper_2406_10707_b200 import workloads as W
    tmp = tempfile.mkdtemp(prefix="lzk_restore_", dir=ROOT)
    try:
        w = W.llama_layer_sample(layers=layers)
        built = lz.build_workload(w.write_spec(os.path.join(tmp, "s.spec")), 0)
        eng = lz.Engine(lz.EngineConfig(checkpoint_root=os.path.join(tmp, "ckpt"),
                                        host_buffer_bytes=int(built.bytes * 1.01) + (64 << 20), device=0),
                        built.topo, built.rank)
        plan = lz.plan_checkpoint(built.topo, built.model, built.step)
        t = eng.capture(plan, built.tree, 1)
        eng.update_barrier(t)
        eng.wait_persisted(t)
        ok, why = eng.commit(built.model, t, lz.ManifestStore(os.path.join(tmp, "manifest.json")))
        assert ok, why
        nbytes = sum(os.path.getsize(f) for f in t.shard_files())
        eng.close()
        del built
        res = {s: [] for s in SETTINGS}
        for r in range(rounds):
            for th, piece in SETTINGS:
                env = dict(os.environ, LZK_ROOT=ROOT, LZK_TMP=tmp, LZK_BYTES=str(nbytes),
                           LZCKPT_READ_THREADS=str(th), LZCKPT_READ_PIECE_MB=str(piece))
                out = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True,
                                     timeout=600)
                line = [l for l in out.stdout.splitlines() if l.startswith("GBPS")]
                if not line:
                    print(out.stdout[-2000:], out.stderr[-2000:], flush=True)
                    raise SystemExit(1)
                v = float(line[0].split()[1])
                res[(th, piece)].append(v)
                print(f"round {r} threads={th} piece={piece}MiB: {v:.3f} GB/s", flush=True)
                time.sleep(pause)
        print(json.dumps({"file_bytes": nbytes, "rounds": rounds,
                          "gbps_median": {f"threads={a} piece={b}MiB": round(statistics.median(v), 3)
                                          for (a, b), v in res.items()}}))
    finally:
        shutil.rmtree(tmp, ignore_errors=True)


if __name__ == "__main__":
    main()
