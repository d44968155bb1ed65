"""Quick GPU end-to-end check: C1 (GPT-2-small shard) through the B200 engine,
whole-file digests vs the reference's golden digests, then restore."""
import os, sys, time, shutil
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_10707_b200 as L
from paper_2406_10707_b200.workloads import gpt2_small

GOLD = {"layers-0-11.ckpt": (248887594, 0x18d06ab61afae34a), "optimizer-0.ckpt": (1493305660, 0xc1f7bf0708955268)}
root = "/tmp/lzk_c1"
shutil.rmtree(root, ignore_errors=True)
spec = gpt2_small().write_spec("/tmp/c1.spec")
t0 = time.time(); w = L.build_workload(spec, 0); print("build", time.time() - t0, w.bytes)
cfg = L.EngineConfig(checkpoint_root=root, host_buffer_bytes=4 << 30, fsync_on_finalize=False)
eng = L.Engine(cfg, w.topo, w.rank)
for step in (1, 2, 3):
    plan = L.plan_checkpoint(w.topo, w.model, step)
    t0 = time.perf_counter(); tk = eng.capture(plan, w.tree, step); t1 = time.perf_counter()
    eng.update_barrier(tk); t2 = time.perf_counter(); eng.wait_persisted(tk); t3 = time.perf_counter()
    print(f"step {step}: capture {1e3*(t1-t0):.2f} ms barrier {1e3*(t2-t1):.2f} ms persisted {1e3*(t3-t0):.1f} ms "
          f"payload {tk.payload_bytes()} -> snapshot {tk.payload_bytes()/(t2-t0)/1e9:.2f} GB/s, persisted {tk.payload_bytes()/(t3-t0)/1e9:.2f} GB/s")
print(eng.snapshot_stats(), eng.counters())
ok = True
for f in tk.shard_files():
    with open(f, "rb") as fh:
        data = fh.read()
    d = L.fnv64(data)
    want = GOLD[os.path.basename(f)]
    print(os.path.basename(f), len(data), hex(d), "OK" if (len(data), d) == want else "MISMATCH")
    ok &= (len(data), d) == want
m = L.ManifestStore(os.path.join(root, "manifest.json"))
m.commit_step(3, L.committed_record(tk, root))
t0 = time.time(); back = eng.restore(m, 3); print("restore", time.time() - t0)
img0 = {l.path: l for l in w.tree.flatten()}
bad = 0
for l in back.flatten():
    a = back.region_at(l.path).clone_bytes() if l.is_region else back.blob_at(l.path)
    b = w.tree.region_at(l.path).clone_bytes() if l.is_region else w.tree.blob_at(l.path)
    bad += a != b
print("restore mismatches", bad, "of", back.leaf_count())
ok &= bad == 0 and back.leaf_count() == w.tree.leaf_count()
print("C1 PARITY", "PASS" if ok else "FAIL")
sys.exit(0 if ok else 1)
