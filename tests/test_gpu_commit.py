"""Commit-time validation on the GPU (validate_rank_files / CommitCoordinator,
reference consolidation.cpp:20-60,160-284): each file streams once, entry
checksums and the whole-file manifest digest are folded by the device FNV
kernels. Checked against the oracle's byte-serial fold of the file bytes and
against the reference's failure reasons (corrupt entry, truncated file)."""
import os

import numpy as np
import pytest

from test_gpu_parity import mixed_tree, small_engine, tiny_model

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gpu(lz):
    assert lz.device_count() > 0, "GPU tests need a CUDA device (no CPU fallback exists)"
    return lz


def persisted(lz, root, step=5):
    eng, topo = small_engine(lz, root)
    tree, _ = mixed_tree(lz, np.random.default_rng(11))
    t = eng.capture(lz.plan_checkpoint(topo, tiny_model(lz), step), tree, step)
    eng.update_barrier(t)
    eng.wait_persisted(t)
    return eng, t


def file_fnv(oracle, path):
    with open(path, "rb") as f:
        return oracle.fnv64(np.frombuffer(f.read(), dtype=np.uint8))


def test_commit_records_gpu_digests(gpu, oracle, tmp_path):
    eng, t = persisted(gpu, tmp_path)
    m = gpu.ManifestStore(str(tmp_path / "manifest.json"))
    ok, why = eng.commit(tiny_model(gpu), t, m)
    assert ok, why
    assert m.is_committed(5)
    import json
    rows = {r["path"]: r for r in json.load(open(tmp_path / "manifest.json"))["steps"][0]["files"]}
    for f in t.shard_files():
        rel = os.path.relpath(f, tmp_path)
        assert rows[rel]["length"] == os.path.getsize(f)
        assert int(rows[rel]["digest"], 16) == file_fnv(oracle, f)
    # the Python helper uses the same device digest
    for rel, n, d in gpu.committed_record(t, str(tmp_path), digest=True):
        assert d == file_fnv(oracle, tmp_path / rel) and n == os.path.getsize(tmp_path / rel)
    eng.close()


def test_commit_rejects_corrupt_and_truncated(gpu, tmp_path):
    eng, t = persisted(gpu, tmp_path)
    f = t.shard_files()[-1]
    h = gpu.read_header(f)
    e = h.entries[-1]
    with open(f, "r+b") as fh:  # flip one payload byte of the last entry
        fh.seek(e.offset + e.length // 2)
        b = fh.read(1)
        fh.seek(e.offset + e.length // 2)
        fh.write(bytes([b[0] ^ 0x5A]))
    m = gpu.ManifestStore(str(tmp_path / "manifest.json"))
    ok, why = eng.commit(tiny_model(gpu), t, m)
    assert not ok and f"checksum mismatch in entry '{e.key}'" in why, why
    assert not m.is_committed(5)
    eng.close()

    root2 = tmp_path / "trunc"
    eng, t = persisted(gpu, root2, step=6)
    f = t.shard_files()[0]
    os.truncate(f, os.path.getsize(f) - 3)
    m = gpu.ManifestStore(str(root2 / "manifest.json"))
    ok, why = eng.commit(tiny_model(gpu), t, m)
    assert not ok and why, why
    assert not m.is_committed(6)
    eng.close()


def test_prepare_vote_and_distributed_commit(gpu, oracle, tmp_path):
    """lzckpt_engine_prepare (this rank's GPU-validated vote) feeding
    commit.distributed_commit (world of one process here; the gloo protocol
    test covers N=2)."""
    from paper_2406_10707_b200.commit import distributed_commit, prepare
    eng, t = persisted(gpu, tmp_path)
    v = prepare(eng, tiny_model(gpu), t)
    assert v["vote"] == "prepared" and v["rank"] == 0 and v["step"] == 5, v
    got = {p: (n, d) for p, n, d in v["files"]}
    for f in t.shard_files():
        assert got[os.path.relpath(f, tmp_path)] == (os.path.getsize(f), file_fnv(oracle, f))
    rec = distributed_commit(eng, tiny_model(gpu), t, str(tmp_path / "manifest.json"))
    assert rec.committed and rec.step == 5
    assert gpu.ManifestStore(str(tmp_path / "manifest.json")).is_committed(5)
    eng.close()
