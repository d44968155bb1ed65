"""Full-size parity at BASELINE.json configs[1] (C2, LLaMA-7B-shaped shard,
107.8 GB, 1164 tensors) through a size-independent property: a checksum of
checksums. The engine captures the whole shard (D2H into the pinned ring) and
its flush hashes every entry exactly as for a real file (hash-only tier: C2
does not fit the box's local disk); the resulting headers - every key,
offset, length and FNV-1a-64 of every byte - must equal the oracle's
headers, computed on the CPU from an independent generation of the same
splitmix64 bytes (oracle.expected_headers). The full 32 layers must run:
on a host that cannot pin the 108 GB shard the largest layer count that fits
is still checked, and the test then XFAILS naming the RAM shortfall, so a
reduced run can never pass as full size."""
import os
import time

import pytest

pytestmark = pytest.mark.gpu


def _mem_available():
    try:
        return next(int(l.split()[1]) * 1024 for l in open("/proc/meminfo") if l.startswith("MemAvailable"))
    except (OSError, StopIteration):
        return 0


def test_c2_fullsize_checksum_of_checksums(lz, oracle, tmp_path):
    from paper_2406_10707_b200.workloads import llama7b_shard
    assert lz.device_count() > 0
    layers = 32
    w = llama7b_shard(layers=layers)
    while w.total_bytes * 1.1 > 0.7 * _mem_available() and layers > 1:
        layers -= 1
        w = llama7b_shard(layers=layers)
    thr = 1 << 20
    t0 = time.time()
    expect = oracle.expected_headers(w, thr, threads=os.cpu_count() or 8)
    t_oracle = time.time() - t0
    built = lz.build_workload(w.write_spec(str(tmp_path / "c2.spec")), 0)
    cfg = lz.EngineConfig(checkpoint_root=str(tmp_path / "ckpt"), host_buffer_bytes=int(built.bytes * 1.01) + (256 << 20),
                          large_leaf_threshold=thr, fsync_on_finalize=False, flush_hash_only=True)
    eng = lz.Engine(cfg, built.topo, built.rank)
    t1 = time.time()
    t = eng.capture(lz.plan_checkpoint(built.topo, built.model, built.step), built.tree, built.step)
    eng.update_barrier(t)
    eng.wait_persisted(t)
    t_engine = time.time() - t1
    got = {os.path.relpath(f, str(tmp_path / "ckpt")): [(e.key, e.offset, e.length, e.checksum) for e in h.entries]
           for f, h in zip(t.shard_files(), eng.ticket_headers(t))}
    assert set(got) == set(expect)
    nentries = 0
    for rel, want in expect.items():
        assert got[rel] == want, (rel, f"layers={layers}")
        nentries += len(want)
    assert t.payload_bytes() == sum(n for hs in expect.values() for _, _, n, _ in hs)
    print(f"C2 layers={layers}: {t.payload_bytes() / 1e9:.1f} GB, {nentries} entries equal to the oracle "
          f"(oracle {t_oracle:.1f} s, engine capture+hash {t_engine:.1f} s)")
    eng.close()
    if layers < 32:
        pytest.xfail(f"host RAM short: MemAvailable {_mem_available() / 1e9:.0f} GB fits {layers} of 32 C2 layers "
                     f"(needs ~{llama7b_shard().total_bytes * 1.1 / 0.7 / 1e9:.0f} GB); the reduced shard matched")
    assert t.payload_bytes() > 107e9 and nentries == 906, "full C2 must have run"


def test_c4_streamed_70b_shard_checksum_of_checksums(lz, oracle, tmp_path):
    """BASELINE.json configs[3]: one rank's ZeRO-style shard of a 70B model
    over dp=8 (10 LLaMA-2-70B decoder layers + embeddings, 372 tensors,
    145.3 GB) streamed through a 32 GiB pinned pool in 1 GiB segments with
    backpressure (the shard and even its optimizer file are larger than the
    pool). Every header entry must equal the oracle's."""
    from paper_2406_10707_b200.workloads import llama70b_shard
    assert lz.device_count() > 0
    w = llama70b_shard()
    pool = 32 << 30
    if pool * 1.5 > _mem_available():
        pytest.xfail(f"host RAM short: MemAvailable {_mem_available() / 1e9:.0f} GB < 48 GiB for the 32 GiB pool")
    thr = 1 << 20
    expect = oracle.expected_headers(w, thr, threads=os.cpu_count() or 8)
    built = lz.build_workload(w.write_spec(str(tmp_path / "c4.spec")), 0)
    cfg = lz.EngineConfig(checkpoint_root=str(tmp_path / "ckpt"), host_buffer_bytes=pool, large_leaf_threshold=thr,
                          fsync_on_finalize=False, flush_hash_only=True, stream_segment_bytes=1 << 30)
    eng = lz.Engine(cfg, built.topo, built.rank)
    t1 = time.time()
    t = eng.capture(lz.plan_checkpoint(built.topo, built.model, built.step), built.tree, built.step)
    eng.update_barrier(t)
    eng.wait_persisted(t)
    t_engine = time.time() - t1
    got = {os.path.relpath(f, str(tmp_path / "ckpt")): [(e.key, e.offset, e.length, e.checksum) for e in h.entries]
           for f, h in zip(t.shard_files(), eng.ticket_headers(t))}
    assert got == expect
    assert t.payload_bytes() > pool * 4
    print(f"C4: {t.payload_bytes() / 1e9:.1f} GB through a {pool >> 30} GiB pool, "
          f"{sum(len(v) for v in expect.values())} entries equal to the oracle ({t_engine:.1f} s)")
    eng.close()
    del built
