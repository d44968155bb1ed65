"""Parity cases for the snapshot path: small workloads that hit the edges the
reference's own tests cover (mixed blobs/regions, inline vs streamed leaves,
per-component path order, byte-granular destinations, zero-size leaves,
multi-rank plans, many small tensors, multi-chunk tensors).

Each case = (Workload, large_leaf_threshold). tests/golden/make_fixtures.py
runs the REFERENCE engine (oracle/_ref/ref_snapshot) on every case and commits
the resulting file sizes + FNV-1a digests to ref_fixtures.json.
"""
from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from paper_2406_10707_b200.workloads import Workload  # noqa: E402


def _plan_sizes(params, layers, bppm, bppo, topo, rank):
    """Shard sizes of plan_checkpoint (reference topology.cpp:100-185),
    restated here so case construction needs no native library."""
    dp, pp, tp = topo[:3]
    rdp, rpp, rtp = rank
    flat = (rdp * pp + rpp) * tp + rtp

    def piece(total, n, i):
        return total // n + (1 if i < total % n else 0)

    first = sum(piece(layers, pp, s) for s in range(rpp))
    cnt = piece(layers, pp, rpp)
    stage = sum(piece(params, layers, l) * bppm for l in range(first, first + cnt))
    out = []
    ls = piece(stage, tp * dp, rdp * tp + rtp)
    if cnt and ls:
        out.append(ls)
    op = piece(params * bppo, dp * pp * tp, flat)
    if op:
        out.append(op)
    return out


def _case(name, params, layers, shards, threshold, topo=(1, 1, 1, 1, 1), rank=(0, 0, 0), bppm=2, bppo=12,
          gen="splitmix64", seed=11, step=1):
    """shards: per plan shard (positional, name order) a (top, [(kind, relpath, size|None)]).
    A None size absorbs the remainder of the shard."""
    sizes = _plan_sizes(params, layers, bppm, bppo, topo, rank)
    assert len(sizes) == len(shards), (name, sizes)
    leaves = []
    for (top, ls), total in zip(shards, sizes):
        fixed = sum(s for _, _, s in ls if s is not None)
        rem = total - fixed
        assert rem >= 0, (name, top, total, fixed)
        for kind, rel, s in ls:
            leaves.append((kind, f"{top}/{rel}", rem if s is None else s))
    w = Workload(name, params, layers, bppm, bppo, leaves, gen=gen, seed=seed, topology=topo, rank=rank, step=step)
    return w, threshold


def all_cases():
    cases = []
    # reference test_engine.cpp:55-63 shape: 4096 params, 4 layers, threshold 4096
    cases.append(_case("mixed", 4096, 4, [
        ("layers", [("r", "block0/w", 5000), ("r", "block1/w", None)]),
        ("optim", [("r", "moments", 40000), ("b", "step", 8), ("b", "extra", None)]),
    ], 4096))
    # per-component ordering traps: a/x < a.b/y < a-b/z ...
    cases.append(_case("order-traps", 20000, 2, [
        ("a_layers", [("r", "a/x", 3001), ("r", "a.b/y", 2999), ("r", "a-b/z", 1), ("r", "a/b/c", 4096),
                      ("b", "A/x", 17), ("r", "a0", 255), ("r", "b/~", None)]),
        ("b_opt", [("r", "z", 100000), ("r", "y/1", 77777), ("r", "y/10", 33333), ("r", "y/2", None)]),
    ], 256))
    # byte-granular destinations: every alignment class, threshold 16
    odd = [1, 2, 3, 7, 15, 16, 17, 31, 33, 63, 65, 127, 129, 4095, 4096, 4097, 65535, 65537,
           (1 << 20) - 1, (1 << 20) + 1, 3 * (1 << 20) + 5]
    cases.append(_case("odd-sizes", 800000, 3, [
        ("a", [("r", f"t{i:02d}", s) for i, s in enumerate(odd[:10])] + [("r", "rest", None)]),
        ("b", [("r", f"u{i:02d}", s) for i, s in enumerate(odd)] + [("b", "blob", 12345), ("r", "rest", None)]),
    ], 16))
    cases.append(_case("all-inline", 3000, 1, [
        ("a", [("r", "w", 5000), ("b", "c", None)]),
        ("b", [("r", "m", 30000), ("r", "v", None)]),
    ], 1 << 30))
    cases.append(_case("threshold-1", 3000, 2, [
        ("a", [("r", "empty_region", 0), ("b", "empty_blob", 0), ("r", "one", 1), ("r", "w", None)]),
        ("b", [("r", "m", 30000), ("b", "s", 3), ("r", "v", None)]),
    ], 1))
    # multi-rank plans (each rank one engine)
    for r in (0, 1):
        cases.append(_case(f"dp2-rank{r}", 100003, 3, [
            ("a", [("r", "w0", 12345), ("r", "w1", None)]),
            ("b", [("r", "m", 500000), ("r", "v", None)]),
        ], 4096, topo=(2, 1, 1, 2, 1), rank=(r, 0, 0), seed=20 + r))
    # BASELINE configs[2]'s plan shape: dp=8, ranks other than 0 (remainder
    # bytes go to the low ranks, topology.cpp:151-182)
    for r in (5, 7):
        cases.append(_case(f"dp8-rank{r}", 800021, 4, [
            ("a", [("r", "w0", 3333), ("r", "w1", None)]),
            ("b", [("r", "m", 400001), ("b", "step", 8), ("r", "v", None)]),
        ], 4096, topo=(8, 1, 1, 8, 1), rank=(r, 0, 0), seed=70 + r))
    cases.append(_case("pp2tp2-rank3", 400009, 5, [
        ("a", [("r", "w", None)]),
        ("b", [("r", "m", 400000), ("b", "step", 8), ("r", "v", None)]),
    ], 4096, topo=(1, 2, 2, 4, 1), rank=(0, 1, 1), seed=31))
    # many small tensors through the gather kernel (> one launch of descriptors)
    small = [("r", f"t{i:05d}", 700 + (i * 37) % 2300) for i in range(3000)]
    cases.append(_case("many-small", 800000, 1, [
        ("a", [("r", "w", None)]),
        ("b", small + [("r", "tail", None)]),
    ], 512, seed=41))
    # multi-chunk tensors (> 64 MiB quantum) + copy-engine class tensors
    cases.append(_case("big", 13_000_000, 2, [
        ("a", [("r", "emb", 3 * (1 << 20) + 7), ("r", "w", None)]),
        ("b", [("r", "m", 67 * (1 << 20) + 3), ("r", "v", 17 * (1 << 20) + 5), ("b", "s", 8), ("r", "rest", None)]),
    ], 1 << 20, seed=51))
    # long, deep and non-ASCII paths: UTF-8 bytes order per component
    # (std::string <), a 600-byte component, 24-level nesting
    deep = "/".join(f"d{i:02d}" for i in range(24))
    cases.append(_case("paths-utf8-deep", 60000, 2, [
        ("a", [("r", "\u03bb/\u00e9t\u00e9", 5000), ("r", "\u03bb/e", 3000), ("r", "Z/\u4e2d\u6587", 4097),
               ("r", "x" * 600, 8191), ("r", deep + "/leaf", 12000), ("b", "\u00ff", 7), ("r", "w", None)]),
        ("b", [("r", "m\u00fcller/\U0001f600", 300000), ("r", "v", None)]),
    ], 4096, seed=61))
    # mt19937_64 generator path (host fill) on a small model
    cases.append(_case("mt-small", 50000, 2, [
        ("a_params", [("r", "w", 60000), ("r", "b", None)]),
        ("b_optim", [("r", "w/fp32", 240000), ("r", "w/exp_avg", 240000), ("r", "rest", None)]),
    ], 65536, gen="mt19937_64", seed=125))
    return cases
