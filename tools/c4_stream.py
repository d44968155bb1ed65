"""BASELINE.json configs[3] at full size on one B200: rank 0 of a dp=8
ZeRO-style 70B plan (145.3 GB: 10 LLaMA-2-70B layers + embeddings) snapshotted
through a 32 GiB pinned pool in 1 GiB segments (streaming + backpressure),
host-memory flush tier. Prints one JSON line.
    python tools/c4_stream.py [pool_GiB]"""
import json
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2406_10707_b200 as lz  # noqa: E402
from paper_2406_10707_b200.workloads import llama70b_shard  # noqa: E402

pool = (int(sys.argv[1]) if len(sys.argv) > 1 else 32) << 30
w = llama70b_shard()
tmp = tempfile.mkdtemp(prefix="lzk_c4_", dir=bench.ROOT)
built = lz.build_workload(w.write_spec(os.path.join(tmp, "c4.spec")), 0)
link = bench.measure_link_ceiling(lz, 0)
plan = lz.plan_checkpoint(built.topo, built.model, built.step)
res = bench.measure_streaming(lz, built, plan, built.bytes, tmp, 0, lambda: None, None, pool=pool, segment=1 << 30)
print(json.dumps({"config": "c4-llama70b rank 0 of dp=8 (configs[3])", "payload_bytes": built.bytes,
                  "tensors": len(w.leaves), "pool_bytes": pool, "segment_bytes": 1 << 30, "gbps": res["gbps"],
                  "frac_of_64": round(res["gbps"] / 64.0, 4), "link_dma_gbps": link["dma_gbps"],
                  "frac_of_measured_dma": round(res["gbps"] / link["dma_gbps"], 4)}))
import shutil  # noqa: E402
shutil.rmtree(tmp, ignore_errors=True)
