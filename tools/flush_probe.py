"""Durable-flush settings on the GPU box's disk: capture -> files fsync'd for
one bounded C2 sample (the e2e workload), per (flush_threads, max_writers,
write_piece). Configurations are interleaved over rounds with a pause in
between, because the disk throttles under sustained writes;
the median per configuration is reported.

    python tools/flush_probe.py [layers] [rounds] [pause_s]
"""
import json
import os
import shutil
import statistics
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2406_10707_b200 as lz  # noqa: E402
from paper_2406_10707_b200 import workloads as W  # noqa: E402

SETS = {  # (flush_threads, max_writers, write_piece MiB)
    "wide": [(0, 0, 32), (0, 1, 64), (0, 2, 32), (0, 2, 64), (0, 4, 32), (0, 1, 128)],
    "writers": [(0, 0, 32), (0, 3, 32), (0, 4, 32), (0, 6, 32), (0, 4, 64)],
}
CONFIGS = SETS[os.environ.get("LZK_FLUSH_SET", "wide")]


def main():
    layers = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    pause = float(sys.argv[3]) if len(sys.argv) > 3 else 8.0
    tmp = tempfile.mkdtemp(prefix="lzk_flush_", dir=ROOT)
    try:
        w = W.llama_layer_sample(layers=layers)
        built = lz.build_workload(w.write_spec(os.path.join(tmp, "s.spec")), 0)
        plan = lz.plan_checkpoint(built.topo, built.model, built.step)
        torch.cuda.synchronize()
        times = {c: [] for c in CONFIGS}
        step = 1
        for r in range(rounds):
            for c in CONFIGS:
                th, wr, piece = c
                root = os.path.join(tmp, "ckpt")
                cfg = lz.EngineConfig(checkpoint_root=root, host_buffer_bytes=int(built.bytes * 1.01) + (64 << 20),
                                      fsync_on_finalize=True, device=0, flush_threads=th, flush_max_writers=wr,
                                      flush_write_piece=piece << 20)
                eng = lz.Engine(cfg, built.topo, built.rank)
                t0 = time.perf_counter()
                t = eng.capture(plan, built.tree, step)
                eng.update_barrier(t)
                eng.wait_persisted(t)
                dt = time.perf_counter() - t0
                payload = t.payload_bytes()
                eng.close()
                step += 1
                shutil.rmtree(root, ignore_errors=True)
                times[c].append(payload / dt / 1e9)
                print(f"round {r} threads={th} writers={wr} piece={piece}MiB: {times[c][-1]:.3f} GB/s", flush=True)
                time.sleep(pause)
        out = {"payload_bytes": payload, "layers": layers, "rounds": rounds, "pause_s": pause,
               "gbps_median": {f"threads={c[0]} writers={c[1]} piece={c[2]}MiB": round(statistics.median(v), 3)
                               for c, v in times.items()}}
        print(json.dumps(out))
    finally:
        shutil.rmtree(tmp, ignore_errors=True)


if __name__ == "__main__":
    main()
