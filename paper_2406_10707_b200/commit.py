"""Multi-process two-phase commit over torch.distributed.

The reference's CommitCoordinator::run_step (proj/core/src/consolidation.cpp:
160-284) runs in one process: ranks are threads, node leaders collect votes,
the coordinator decides. A real job has one process per GPU, so here:

  phase one   every rank calls ``prepare`` (lzckpt_engine_prepare: wait until
              its capture is persisted, then validate its own files on its GPU
              -- header, extent, entry checksums and the whole-file manifest
              digest, each file read once);
  votes       travel to rank 0 (``gather_object``);
  decision    rank 0 decides as the reference coordinator does (``decide``):
              committed iff every rank prepared; otherwise aborted with the
              first failing rank blamed as "rank R: <detail>";
  durability  on commit rank 0 writes the manifest (files sorted by path,
              tmp + rename) BEFORE anyone learns the decision;
  phase two   the decision is broadcast to every rank.

A rank that never answers surfaces as the process group's timeout (the
reference's per-step vote deadline is the group timeout here).
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import json
from typing import Callable, List, Optional, Sequence

from . import lzckpt as _lz
from ._native import lib


@dataclasses.dataclass
class CommitRecord:
    step: int
    committed: bool
    reason: str = ""
    problem_ranks: List[int] = dataclasses.field(default_factory=list)
    files: List[tuple] = dataclasses.field(default_factory=list)  # (path, length, digest), rank 0 only


def prepare(engine: "_lz.Engine", model: "_lz.ModelSpec", ticket: "_lz.CaptureTicket") -> dict:
    """This rank's vote (EngineCommitParticipant::prepare): {"rank", "step",
    "vote": "prepared"|"failed", "detail", "files": [[path, length, digest]]}."""
    need = C.c_uint64()
    cap = 1 << 16
    while True:
        buf = C.create_string_buffer(cap)
        _lz._check(lib.lzckpt_engine_prepare(engine._h, C.byref(model._c()), ticket._h, buf, cap, C.byref(need)))
        if need.value <= cap:
            return json.loads(buf.value.decode())
        cap = int(need.value)


def decide(votes: Sequence[Optional[dict]], world: int) -> CommitRecord:
    """The coordinator's decision over one vote per rank (None = no answer),
    as in consolidation.cpp:229-283."""
    step = next((v["step"] for v in votes if v), 0)
    problems, reason, files = [], "", []
    for r in range(world):
        v = votes[r] if r < len(votes) else None
        if v is None:
            problems.append(r)
            reason = reason or f"rank {r} did not answer before the timeout"
        elif v["vote"] != "prepared":
            problems.append(v.get("rank", r))
            reason = reason or f"rank {v.get('rank', r)}: {v['detail']}"
        else:
            files.extend(tuple(f) for f in v["files"])
    if problems:
        return CommitRecord(step, False, reason, sorted(problems))
    return CommitRecord(step, True, files=sorted(files))


def distributed_commit(engine: "_lz.Engine", model: "_lz.ModelSpec", ticket: "_lz.CaptureTicket",
                       manifest_path: str, group=None,
                       prepare_fn: Optional[Callable[[], dict]] = None) -> CommitRecord:
    """Two-phase commit of one step across all ranks of ``group`` (default:
    the world). Every rank calls it with its own engine and ticket; every
    rank returns the same CommitRecord. ``prepare_fn`` replaces the GPU
    validation (tests of the protocol on CPU)."""
    import torch.distributed as dist
    vote = prepare_fn() if prepare_fn else prepare(engine, model, ticket)
    if not dist.is_available() or not dist.is_initialized():
        votes, world, rank = [vote], 1, 0
    else:
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        votes = [None] * world if rank == 0 else None
        dist.gather_object(vote, votes, dst=dist.get_global_rank(group, 0) if group else 0, group=group)
    out = [None]
    if rank == 0:
        rec = decide(votes, world)
        if rec.committed:
            m = _lz.ManifestStore(manifest_path)
            m.commit_step(rec.step, [(p, int(n), int(d)) for p, n, d in rec.files])  # durable before anyone learns
        out[0] = CommitRecord(rec.step, rec.committed, rec.reason, rec.problem_ranks)
    if world > 1:
        dist.broadcast_object_list(out, src=dist.get_global_rank(group, 0) if group else 0, group=group)
    return out[0]
