"""gather-kernel grid size vs throughput per size class (smallest grid that
saturates the host link = least SM theft from training)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_10707_b200 as lz
from paper_2406_10707_b200.workloads import sweep_class
for size, count in [(4096, 10000), (65536, 10000), (1 << 20, 1024), (64 << 20, 16)]:
    w = sweep_class(size, size * count)
    built = lz.build_workload(w.write_spec(f"/tmp/cs_{size}.spec"), 0)
    cfg = lz.EngineConfig(checkpoint_root="/tmp/cs", host_buffer_bytes=int(built.bytes * 1.05) + (64 << 20),
                          large_leaf_threshold=min(4096, size), fsync_on_finalize=False, flush_discard=True,
                          force_kernel=True)
    eng = lz.Engine(cfg, built.topo, built.rank)
    plan = lz.plan_checkpoint(built.topo, built.model, built.step)
    row = {"class": size}
    for ctas in (2, 4, 8, 12, 16, 32):
        eng.set_copy_variant(force_kernel=True, kernel_ctas=ctas)
        d = []
        for s in range(4):
            t = eng.capture(plan, built.tree, s + 1)
            eng.update_barrier(t)
            eng.wait_persisted(t)
            if s:
                d.append(eng.ticket_device_ms(t))
        row[ctas] = round(t.payload_bytes() / (sum(d) / len(d) * 1e-3) / 1e9, 2)
    print(json.dumps(row), flush=True)
    eng.close()
