"""Python mirror of the lzckpt engine API over the C ABI (include/lzckpt_c.h).

Class, method and exception names follow the reference C++ API
(/root/reference/proj/core/include/lzckpt/*.hpp) so code and tests read the
same: ``StateTree.set_region``, ``Engine.capture / update_barrier /
wait_persisted / drain / restore``, ``TornSnapshot`` ... Every call goes
through liblzckpt_b200.so; nothing here moves or hashes payload bytes.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
import sys
from typing import Callable, Iterable, List, Optional, Sequence, Tuple

from . import _native as N

lib = N.lib
dev = N.dev

# ---------------------------------------------------------------------------
# exceptions (reference errors.hpp:8-82), one per C-ABI status code


class Error(RuntimeError):
    pass


class ConfigError(Error):
    pass


class SizeExceedsCapacity(ConfigError):
    pass


class WaitTimeout(Error):
    pass


class IllegalTransition(Error):
    pass


class TornSnapshot(Error):
    pass


class DuplicatePath(Error):
    pass


class FormatError(Error):
    pass


class BadMagic(FormatError):
    pass


class TruncatedFile(FormatError):
    pass


class ChecksumMismatch(FormatError):
    pass


class NotCommitted(Error):
    pass


class CorruptManifest(Error):
    pass


class IoError(Error):
    pass


class DeviceError(Error):
    pass


class InvalidArgument(Error, ValueError):
    pass


_CODES = {1: Error, 2: ConfigError, 3: SizeExceedsCapacity, 4: WaitTimeout, 5: IllegalTransition,
          6: TornSnapshot, 7: DuplicatePath, 8: FormatError, 9: BadMagic, 10: TruncatedFile,
          11: ChecksumMismatch, 12: NotCommitted, 13: CorruptManifest, 14: IoError, 15: DeviceError,
          16: InvalidArgument}


def _check(rc: int) -> None:
    if rc != 0:
        msg = lib.lzckpt_last_error().decode(errors="replace")
        raise _CODES.get(rc, Error)(msg)


def _buf(data) -> Tuple[object, int]:
    """(pointer, length) for bytes-like input without copying when possible."""
    if isinstance(data, (bytes, bytearray)):
        b = data if isinstance(data, bytearray) else bytearray(data)
        return (C.c_char * len(b)).from_buffer(b) if len(b) else None, len(b)
    mv = memoryview(data).cast("B")
    b = bytearray(mv)
    return (C.c_char * len(b)).from_buffer(b) if len(b) else None, len(b)


def fnv64(data) -> int:
    p, n = _buf(data)
    return lib.lzckpt_fnv1a64(p, n)


# ---------------------------------------------------------------------------
# topology / plan (reference topology.hpp:12-110)


@dataclasses.dataclass
class ParallelTopology:
    dp: int = 1
    pp: int = 1
    tp: int = 1
    gpus_per_node: int = 4
    node_count: int = 1

    def ranks(self) -> int:
        return self.dp * self.pp * self.tp

    def _c(self) -> N.Topology:
        return N.Topology(self.dp, self.pp, self.tp, self.gpus_per_node, self.node_count)


@dataclasses.dataclass
class RankCoord:
    dp: int = 0
    pp: int = 0
    tp: int = 0


def flat_rank(topo: ParallelTopology, r: RankCoord) -> int:
    return (r.dp * topo.pp + r.pp) * topo.tp + r.tp


@dataclasses.dataclass
class ModelSpec:
    name: str = ""
    param_count: int = 0
    layer_count: int = 1
    hidden_dim: int = 0
    bytes_per_param_model: int = 2
    bytes_per_param_optimizer: int = 12

    def _c(self) -> N.ModelSpecC:
        return N.ModelSpecC(self.param_count, self.layer_count, self.hidden_dim,
                            self.bytes_per_param_model, self.bytes_per_param_optimizer)


@dataclasses.dataclass
class ShardDescriptor:
    shard_id: int
    kind: str  # "layers" | "optimizer"
    first_layer: int
    layer_count: int
    partition: int
    size_bytes: int
    owner: RankCoord
    filename: str


class CheckpointPlan:
    """plan_checkpoint(topo, model, step) (reference topology.cpp:100-185)."""

    def __init__(self, topo: ParallelTopology, model: ModelSpec, step: int):
        self.topo, self.model, self.step = topo, model, step
        self._shards = [self._rank_shards(r) for r in range(topo.ranks())]

    def _rank_shards(self, rank: int) -> List[ShardDescriptor]:
        arr = (N.ShardC * 4)()
        n = C.c_uint32()
        _check(lib.lzckpt_plan_shards(C.byref(self.topo._c()), C.byref(self.model._c()), rank, arr, 4,
                                      C.byref(n)))
        return [ShardDescriptor(s.shard_id, "layers" if s.kind == 0 else "optimizer", s.first_layer,
                                s.layer_count, s.partition, s.size_bytes,
                                RankCoord(s.owner_dp, s.owner_pp, s.owner_tp), s.filename.decode())
                for s in arr[: n.value]]

    def shards(self, rank) -> List[ShardDescriptor]:
        if isinstance(rank, RankCoord):
            rank = flat_rank(self.topo, rank)
        return self._shards[rank]

    def total_bytes(self) -> int:
        return sum(s.size_bytes for r in self._shards for s in r)

    def rank_bytes(self, rank: int) -> int:
        return sum(s.size_bytes for s in self._shards[rank])


def plan_checkpoint(topo: ParallelTopology, model: ModelSpec, step: int) -> CheckpointPlan:
    return CheckpointPlan(topo, model, step)


# ---------------------------------------------------------------------------
# device regions (reference transfer_engine.hpp:24-43)


class DeviceRegion:
    """HBM allocation with a version counter. ``DeviceRegion(n)`` zero-fills,
    ``DeviceRegion(bytes)`` uploads, ``DeviceRegion.wrap(tensor)`` views a
    torch CUDA tensor's storage without copying."""

    def __init__(self, size_or_bytes=0, device: int = -1, _handle=None, _keepalive=None):
        self._keep = _keepalive
        if _handle is not None:
            self._h = _handle
            return
        h = C.c_void_p()
        if isinstance(size_or_bytes, int):
            _check(lib.lzckpt_region_create(device, size_or_bytes, C.byref(h)))
        else:
            p, n = _buf(size_or_bytes)
            _check(lib.lzckpt_region_from_host(device, p, n, C.byref(h)))
        self._h = h

    @classmethod
    def wrap(cls, tensor, device: Optional[int] = None) -> "DeviceRegion":
        """Register a contiguous CUDA tensor (its bytes, in storage order)."""
        if not tensor.is_cuda or not tensor.is_contiguous():
            raise InvalidArgument("DeviceRegion.wrap needs a contiguous CUDA tensor")
        h = C.c_void_p()
        d = tensor.device.index if device is None else device
        _check(lib.lzckpt_region_wrap(d, tensor.data_ptr(), tensor.numel() * tensor.element_size(),
                                      C.byref(h)))
        return cls(_handle=h, _keepalive=tensor)

    @classmethod
    def wrap_ptr(cls, device: int, ptr: int, size: int) -> "DeviceRegion":
        h = C.c_void_p()
        _check(lib.lzckpt_region_wrap(device, ptr, size, C.byref(h)))
        return cls(_handle=h)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib.lzckpt_region_release(h)
            self._h = None

    def size(self) -> int:
        return lib.lzckpt_region_size(self._h)

    def version(self) -> int:
        return lib.lzckpt_region_version(self._h)

    @property
    def device_ptr(self) -> int:
        return lib.lzckpt_region_device_ptr(self._h) or 0

    @property
    def device(self) -> int:
        return lib.lzckpt_region_device(self._h)

    def read_chunk(self, offset: int, n: int) -> bytes:
        out = (C.c_char * max(n, 1))()
        _check(lib.lzckpt_region_read(self._h, offset, out, n))
        return bytes(out.raw[:n])

    def clone_bytes(self) -> bytes:
        return self.read_chunk(0, self.size())

    def write(self, offset: int, data) -> None:
        p, n = _buf(data)
        _check(lib.lzckpt_region_write(self._h, offset, p, n))

    def mutate(self, fn: Callable[[bytearray], None]) -> None:
        """Reference semantics: one call, one version bump. ``fn`` edits a
        host image of the region in place (staged D2H -> fn -> H2D)."""
        img = bytearray(self.clone_bytes())
        fn(img)
        p, n = _buf(img)
        _check(lib.lzckpt_region_mutate(self._h, p, n))

    def bump_version(self) -> None:
        _check(lib.lzckpt_region_bump_version(self._h))


# ---------------------------------------------------------------------------
# state tree (reference state_tree.hpp:19-79)


@dataclasses.dataclass
class FlatLeaf:
    path: str
    is_region: bool
    size: int


class StateTree:
    META_KEY = "__meta__"

    def __init__(self, _handle=None):
        if _handle is None:
            _handle = C.c_void_p()
            _check(lib.lzckpt_tree_create(C.byref(_handle)))
        self._h = _handle
        self._regions = []  # keep wrapped tensors alive

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib.lzckpt_tree_destroy(h)
            self._h = None

    def set_region(self, path: str, region: DeviceRegion) -> None:
        _check(lib.lzckpt_tree_set_region(self._h, path.encode(), region._h))
        self._regions.append(region)

    def set_blob(self, path: str, data) -> None:
        p, n = _buf(data)
        _check(lib.lzckpt_tree_set_blob(self._h, path.encode(), p, n))

    def leaf_count(self) -> int:
        return lib.lzckpt_tree_leaf_count(self._h)

    def total_leaf_bytes(self) -> int:
        return lib.lzckpt_tree_total_bytes(self._h)

    def flatten(self) -> List[FlatLeaf]:
        out = []
        buf = C.create_string_buffer(1 << 16)
        isr, sz = C.c_int(), C.c_uint64()
        for i in range(self.leaf_count()):
            _check(lib.lzckpt_tree_leaf(self._h, i, buf, len(buf), C.byref(isr), C.byref(sz)))
            out.append(FlatLeaf(buf.value.decode(), bool(isr.value), sz.value))
        return out

    def region_at(self, path: str) -> DeviceRegion:
        h = C.c_void_p()
        _check(lib.lzckpt_tree_region_at(self._h, path.encode(), C.byref(h)))
        return DeviceRegion(_handle=h)

    def blob_at(self, path: str) -> bytes:
        n = C.c_uint64()
        _check(lib.lzckpt_tree_blob_at(self._h, path.encode(), None, 0, C.byref(n)))
        out = (C.c_char * max(n.value, 1))()
        _check(lib.lzckpt_tree_blob_at(self._h, path.encode(), out, n.value, C.byref(n)))
        return bytes(out.raw[: n.value])

    def image(self) -> dict:
        """{path: (is_region, bytes)} — test helper (reference test_engine.cpp image_of)."""
        return {l.path: (l.is_region, self.region_at(l.path).clone_bytes() if l.is_region
                         else self.blob_at(l.path)) for l in self.flatten()}


# ---------------------------------------------------------------------------
# shard file format (reference format.hpp:15-72)


@dataclasses.dataclass
class HeaderEntry:
    key: str
    offset: int = 0
    length: int = 0
    checksum: int = 0


@dataclasses.dataclass
class CheckpointFileHeader:
    entries: List[HeaderEntry]
    format_version: int = 1

    def serialized_size(self) -> int:
        return 24 + sum(28 + len(e.key.encode()) for e in self.entries)

    def payload_end(self) -> int:
        return max([self.serialized_size()] + [e.offset + e.length for e in self.entries])

    def find(self, key: str) -> Optional[HeaderEntry]:
        for e in self.entries:
            if e.key == key:
                return e
        return None


def _entries_c(h: CheckpointFileHeader):
    keys = [e.key.encode() for e in h.entries]
    arr = (N.HeaderEntryC * max(len(keys), 1))()
    bufs = [C.create_string_buffer(k, len(k) + 1) for k in keys]
    for i, e in enumerate(h.entries):
        arr[i] = N.HeaderEntryC(C.cast(bufs[i], C.c_void_p), len(keys[i]), e.offset, e.length, e.checksum)
    return arr, bufs


def serialize_header(h: CheckpointFileHeader) -> bytes:
    arr, _keep = _entries_c(h)
    need = C.c_uint64()
    _check(lib.lzckpt_header_serialize(arr, len(h.entries), h.format_version, None, 0, C.byref(need)))
    out = (C.c_char * need.value)()
    _check(lib.lzckpt_header_serialize(arr, len(h.entries), h.format_version, out, need.value, C.byref(need)))
    return bytes(out.raw)


def _from_handle(hh) -> CheckpointFileHeader:
    try:
        ents = []
        e = N.HeaderEntryC()
        for i in range(lib.lzckpt_header_count(hh)):
            _check(lib.lzckpt_header_entry_at(hh, i, C.byref(e)))
            key = C.string_at(e.key, e.key_len).decode(errors="surrogateescape")
            ents.append(HeaderEntry(key, e.offset, e.length, e.checksum))
        return CheckpointFileHeader(ents, lib.lzckpt_header_version(hh))
    finally:
        lib.lzckpt_header_destroy(hh)


def parse_header(data) -> CheckpointFileHeader:
    p, n = _buf(data)
    hh = C.c_void_p()
    _check(lib.lzckpt_header_parse(p, n, C.byref(hh)))
    return _from_handle(hh)


def read_header(path) -> CheckpointFileHeader:
    hh = C.c_void_p()
    _check(lib.lzckpt_file_read_header(os.fspath(path).encode(), C.byref(hh)))
    return _from_handle(hh)


def validate_entries(path, header: CheckpointFileHeader) -> List[str]:
    raw = serialize_header(header)
    hh = C.c_void_p()
    _check(lib.lzckpt_header_parse(raw, len(raw), C.byref(hh)))
    try:
        out = C.create_string_buffer(1 << 20)
        nbad = C.c_uint32()
        _check(lib.lzckpt_file_validate(os.fspath(path).encode(), hh, out, len(out), C.byref(nbad)))
        return out.value.decode().split("\n") if nbad.value else []
    finally:
        lib.lzckpt_header_destroy(hh)


def read_entry(path, header: CheckpointFileHeader, key: str) -> bytes:
    e = header.find(key)
    if e is None:
        raise FormatError(f"{path}: no entry named '{key}'")
    with open(path, "rb") as f:
        f.seek(e.offset)
        b = f.read(e.length)
    if len(b) != e.length:
        raise TruncatedFile(f"{path}: short read for entry '{key}'")
    return b


# ---------------------------------------------------------------------------
# ring core (reference ring_core.hpp:31-68) — pure state machine


class RingCore:
    STATES = ("Reserved", "Filled", "Flushing", "Free")

    def __init__(self, capacity: int):
        self._h = C.c_void_p()
        _check(lib.lzckpt_ring_create(capacity, C.byref(self._h)))
        self.capacity = capacity

    def __del__(self):
        if getattr(self, "_h", None):
            lib.lzckpt_ring_destroy(self._h)
            self._h = None

    def try_reserve(self, size: int, ticket: int = 0) -> Optional[Tuple[int, int]]:
        i, o = C.c_uint64(), C.c_uint64()
        _check(lib.lzckpt_ring_try_reserve(self._h, size, ticket, C.byref(i), C.byref(o)))
        return None if i.value == 0 else (i.value, o.value)

    def mark_filled(self, sid: int):
        _check(lib.lzckpt_ring_mark_filled(self._h, sid))

    def begin_flush(self, sid: int):
        _check(lib.lzckpt_ring_begin_flush(self._h, sid))

    def release(self, sid: int):
        _check(lib.lzckpt_ring_release(self._h, sid))

    def live_bytes(self) -> int:
        return lib.lzckpt_ring_live_bytes(self._h)

    def live_segments(self) -> int:
        return lib.lzckpt_ring_live_segments(self._h)

    def released_bytes(self) -> int:
        return lib.lzckpt_ring_released_bytes(self._h)

    def segment(self, sid: int) -> Tuple[int, int, str]:
        o, l, s = C.c_uint64(), C.c_uint64(), C.c_int()
        _check(lib.lzckpt_ring_segment(self._h, sid, C.byref(o), C.byref(l), C.byref(s)))
        return o.value, l.value, self.STATES[s.value]


# ---------------------------------------------------------------------------
# manifest (reference manifest.hpp:29-49)


class ManifestStore:
    def __init__(self, path):
        self.path = os.fspath(path)
        self._h = C.c_void_p()
        _check(lib.lzckpt_manifest_open(self.path.encode(), C.byref(self._h)))

    def __del__(self):
        if getattr(self, "_h", None):
            lib.lzckpt_manifest_destroy(self._h)
            self._h = None

    def commit_step(self, step: int, files: Sequence[Tuple[str, int, int]]) -> None:
        """files: (relative_path, length, whole-file digest)."""
        n = len(files)
        paths = (C.c_char_p * max(n, 1))(*[f[0].encode() for f in files])
        lens = (C.c_uint64 * max(n, 1))(*[f[1] for f in files])
        digs = (C.c_uint64 * max(n, 1))(*[f[2] for f in files])
        _check(lib.lzckpt_manifest_commit_step(self._h, step, paths, lens, digs, n))

    def is_committed(self, step: int) -> bool:
        return bool(lib.lzckpt_manifest_is_committed(self._h, step))

    def latest_committed(self) -> Optional[int]:
        has, step = C.c_int(), C.c_uint64()
        _check(lib.lzckpt_manifest_latest(self._h, C.byref(has), C.byref(step)))
        return step.value if has.value else None


# ---------------------------------------------------------------------------
# engine (reference engine.hpp:32-147)


@dataclasses.dataclass
class EngineConfig:
    checkpoint_root: str = ""
    host_buffer_bytes: int = 16_000_000_000
    copy_bandwidth_Bps: float = 0.0   # reference ThrottledChannel.bandwidth_Bps (0: unpaced)
    chunk_quantum: int = 64 << 20
    storage_bandwidth_Bps: float = 0.0
    fsync_on_finalize: bool = True
    flush_threads: int = 0
    large_leaf_threshold: int = 1 << 20
    reserve_timeout_ms: int = 60_000
    device: int = -1
    ce_threshold: int = 2 << 20
    kernel_ctas: int = 4
    group_bytes: int = 256 << 20
    force_kernel: bool = False
    force_copy_engine: bool = False
    hugepages: bool = True
    flush_discard: bool = False
    stream_segment_bytes: int = 0
    flush_hash_only: bool = False
    # uplink relay between the ranks of one node (EngineConfig::Relay)
    relay_serve_socket: str = ""   # helper: serve relay requests on this Unix socket
    relay_staging_bytes: int = 1 << 30
    relay_ctas: int = 4
    relay_peer_socket: str = ""    # owner: delegate to the helper listening here
    relay_share: float = 0.0       # fraction of each shard file's payload
    relay_min_entry: int = 64 << 20
    relay_kernel_route: bool = False  # helper: SM gather kernel instead of copy engines
    flush_max_writers: int = 3  # concurrent pwrite jobs (0: bounded by flush_threads only)
    flush_write_piece: int = 32 << 20  # max bytes per pwrite job

    _STRINGS = ("checkpoint_root", "relay_serve_socket", "relay_peer_socket")

    def _c(self) -> N.EngineConfigC:
        c = N.EngineConfigC()
        lib.lzckpt_engine_config_defaults(C.byref(c))
        self._keep = [os.fspath(getattr(self, k)).encode() for k in self._STRINGS]
        c.checkpoint_root, c.relay_serve_socket, c.relay_peer_socket = self._keep
        for f in dataclasses.fields(self):
            if f.name in self._STRINGS:
                continue
            v = getattr(self, f.name)
            setattr(c, f.name, int(v) if isinstance(v, bool) else v)
        return c


TICKET_STATUS = ("in-flight", "host-resident", "persisted", "failed")


class CaptureTicket:
    def __init__(self, handle):
        self._h = handle

    def __del__(self):
        if getattr(self, "_h", None):
            lib.lzckpt_ticket_release(self._h)
            self._h = None

    def id(self) -> int:
        return lib.lzckpt_ticket_id(self._h)

    def step(self) -> int:
        return lib.lzckpt_ticket_step(self._h)

    def status(self) -> str:
        return TICKET_STATUS[lib.lzckpt_ticket_status(self._h)]

    def torn(self) -> bool:
        return bool(lib.lzckpt_ticket_torn(self._h))

    def payload_bytes(self) -> int:
        return lib.lzckpt_ticket_payload_bytes(self._h)

    def shard_files(self) -> List[str]:
        buf = C.create_string_buffer(4096)
        out = []
        for i in range(lib.lzckpt_ticket_file_count(self._h)):
            _check(lib.lzckpt_ticket_file(self._h, i, buf, len(buf)))
            out.append(buf.value.decode())
        return out

    def failure_reason(self) -> str:
        buf = C.create_string_buffer(4096)
        _check(lib.lzckpt_ticket_failure_reason(self._h, buf, len(buf)))
        return buf.value.decode()


@dataclasses.dataclass
class Counters:
    captures: int
    bytes_captured: int
    capture_seconds: float
    barrier_seconds: float
    last_capture_seconds: float
    last_barrier_seconds: float


class _CurrentStream:
    """Default producer for Engine.capture: torch's current CUDA stream on the
    engine's device (when torch has initialised CUDA in this process)."""

    def __repr__(self):
        return "CURRENT_STREAM"


CURRENT_STREAM = _CurrentStream()


def _producer(stream, device: int):
    """(ordered, cudaStream_t) for a capture's producer argument.

    CURRENT_STREAM -> torch.cuda.current_stream(device) if torch has set up
    CUDA here, else unordered (no torch work can be pending); None ->
    unordered, the reference call; a torch.cuda.Stream or a raw int handle
    (0 = the legacy default stream) -> ordered after that stream."""
    if stream is CURRENT_STREAM:
        torch = sys.modules.get("torch")
        if torch is None or not torch.cuda.is_initialized():
            return False, None
        d = torch.cuda.current_device() if device < 0 else device
        return True, torch.cuda.current_stream(d).cuda_stream
    if stream is None:
        return False, None
    return True, int(getattr(stream, "cuda_stream", stream))


class Engine:
    def __init__(self, config: EngineConfig, topo: ParallelTopology, rank: RankCoord):
        self.config, self.topo, self.rank = config, topo, rank
        self._cfg = config._c()
        self._h = C.c_void_p()
        _check(lib.lzckpt_engine_create(C.byref(self._cfg), C.byref(topo._c()), rank.dp, rank.pp, rank.tp,
                                        C.byref(self._h)))

    def close(self):
        if getattr(self, "_h", None):
            lib.lzckpt_engine_destroy(self._h)
            self._h = None

    __del__ = close

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def capture(self, plan: CheckpointPlan, state: StateTree, step: int,
                producer_stream=CURRENT_STREAM) -> CaptureTicket:
        """Engine::capture. The snapshot is ordered on the device after the work
        already queued on `producer_stream` (default: torch's current stream),
        so it never reads a tensor the trainer is still writing; the host does
        not wait. producer_stream=None is the reference call (inline leaves
        cloned synchronously, no producer ordering)."""
        h = C.c_void_p()
        ordered, handle = _producer(producer_stream, self.config.device)
        if ordered:
            _check(lib.lzckpt_engine_capture_on_stream(self._h, C.byref(plan.model._c()), state._h, step, handle,
                                                       C.byref(h)))
        else:
            _check(lib.lzckpt_engine_capture(self._h, C.byref(plan.model._c()), state._h, step, C.byref(h)))
        return CaptureTicket(h)

    def ticket_headers(self, t: CaptureTicket) -> List[CheckpointFileHeader]:
        out = []
        for i in range(lib.lzckpt_ticket_file_count(t._h)):
            hh = C.c_void_p()
            _check(lib.lzckpt_engine_ticket_header(self._h, t._h, i, C.byref(hh)))
            out.append(_from_handle(hh))
        return out

    def capture_file(self, path, state: StateTree, step: int, producer_stream=CURRENT_STREAM) -> CaptureTicket:
        h = C.c_void_p()
        ordered, handle = _producer(producer_stream, self.config.device)
        if ordered:
            _check(lib.lzckpt_engine_capture_file_on_stream(self._h, os.fspath(path).encode(), state._h, step,
                                                            handle, C.byref(h)))
        else:
            _check(lib.lzckpt_engine_capture_file(self._h, os.fspath(path).encode(), state._h, step, C.byref(h)))
        return CaptureTicket(h)

    def restore_file(self, path, into: Optional[StateTree] = None) -> StateTree:
        h = C.c_void_p()
        _check(lib.lzckpt_engine_restore_file(self._h, os.fspath(path).encode(), into._h if into else None,
                                              C.byref(h)))
        return StateTree(_handle=h)

    def update_barrier(self, t: CaptureTicket) -> None:
        _check(lib.lzckpt_engine_update_barrier(self._h, t._h))

    def update_barrier_on_stream(self, t: CaptureTicket, cuda_stream: int) -> None:
        _check(lib.lzckpt_engine_update_barrier_on_stream(self._h, t._h, cuda_stream))

    def wait_persisted(self, t: CaptureTicket) -> None:
        _check(lib.lzckpt_engine_wait_persisted(self._h, t._h))

    def drain(self) -> None:
        _check(lib.lzckpt_engine_drain(self._h))

    def restore(self, manifest: ManifestStore, step: int) -> StateTree:
        h = C.c_void_p()
        _check(lib.lzckpt_engine_restore(self._h, manifest._h, step, C.byref(h)))
        return StateTree(_handle=h)

    def restore_into(self, manifest: ManifestStore, step: int, tree: StateTree) -> None:
        _check(lib.lzckpt_engine_restore_into(self._h, manifest._h, step, tree._h))

    def commit(self, model: ModelSpec, t: CaptureTicket, manifest: ManifestStore) -> Tuple[bool, str]:
        """Two-phase commit of a persisted capture (reference
        CommitCoordinator::run_step, consolidation.cpp:160-284): files are
        validated and their whole-file digests recorded, each file read once
        and hashed on the GPU. Returns (committed, reason)."""
        ok = C.c_int()
        reason = C.create_string_buffer(1024)
        _check(lib.lzckpt_engine_commit(self._h, C.byref(model._c()), t._h, manifest._h, C.byref(ok), reason, 1024))
        return bool(ok.value), reason.value.decode(errors="replace")

    def numa_node(self) -> int:
        """NUMA node of this engine's pinned ring and threads (-1: none)."""
        return lib.lzckpt_engine_numa_node(self._h)

    def set_relay(self, peer_socket: str, share: float) -> None:
        """Delegate `share` of each shard file's payload to the helper serving
        `peer_socket` (share 0: off). Call between captures."""
        _check(lib.lzckpt_engine_set_relay(self._h, os.fspath(peer_socket).encode(), share))

    def relay_stats(self) -> dict:
        """Uplink relay counters: bytes delegated to the helper (owner), bytes
        and requests relayed for owners (helper)."""
        a, b, c = C.c_uint64(), C.c_uint64(), C.c_uint64()
        _check(lib.lzckpt_engine_relay_stats(self._h, C.byref(a), C.byref(b), C.byref(c)))
        return {"delegated_bytes": a.value, "served_bytes": b.value, "served_requests": c.value}

    def counters(self) -> Counters:
        c = N.CountersC()
        _check(lib.lzckpt_engine_counters(self._h, C.byref(c)))
        return Counters(c.captures, c.bytes_captured, c.capture_seconds, c.barrier_seconds,
                        c.last_capture_seconds, c.last_barrier_seconds)

    def snapshot_stats(self) -> dict:
        s = N.SnapshotStatsC()
        _check(lib.lzckpt_engine_snapshot_stats(self._h, C.byref(s)))
        return {f[0]: getattr(s, f[0]) for f in N.SnapshotStatsC._fields_}

    def flush_stats(self) -> Tuple[int, int]:
        b, f = C.c_uint64(), C.c_uint64()
        _check(lib.lzckpt_engine_flush_stats(self._h, C.byref(b), C.byref(f)))
        return b.value, f.value

    def ticket_device_ms(self, t: CaptureTicket) -> float:
        return lib.lzckpt_engine_ticket_device_ms(self._h, t._h)

    def set_copy_variant(self, ce_threshold: int = 2 << 20, force_kernel: bool = False,
                         force_copy_engine: bool = False, kernel_ctas: int = 0, group_bytes: int = 0) -> None:
        _check(lib.lzckpt_engine_set_copy_variant(self._h, ce_threshold, int(force_kernel), int(force_copy_engine),
                                                  kernel_ctas, group_bytes))

    @property
    def snapshot_stream(self) -> int:
        return lib.lzckpt_engine_snapshot_stream(self._h) or 0


def committed_record(ticket: CaptureTicket, root: str, digest: bool = False,
                     device: int = 0) -> List[Tuple[str, int, int]]:
    """Manifest rows for a persisted ticket (reference test_engine.cpp:73-84);
    with digest=True the whole-file FNV-1a the manifest records, computed on
    the GPU (lzckpt_file_digest)."""
    rows = []
    for f in ticket.shard_files():
        d = 0
        n = os.path.getsize(f)
        if digest:
            ln, dg = C.c_uint64(), C.c_uint64()
            _check(lib.lzckpt_file_digest(os.fspath(f).encode(), device, C.byref(ln), C.byref(dg)))
            n, d = ln.value, dg.value
        rows.append((os.path.relpath(f, root), n, d))
    return rows


def trim_caches() -> None:
    """Free the stream windows restore/commit keep pooled between calls
    (3 x 512 MiB pinned + 3 x 512 MiB HBM per device)."""
    lib.lzckpt_trim_caches()


def device_numa_node(device: int = 0) -> int:
    """NUMA node of the GPU's PCI function; -1 when the host reports none."""
    n = C.c_int(-1)
    _dev_check(dev.lzk_device_numa_node(device, C.byref(n)))
    return n.value


def numa_node_count() -> int:
    return lib.lzckpt_numa_node_count()


def numa_page_nodes(address: int, length: int, stride: int = 4096) -> List[int]:
    """Node holding each page of [address, address+length) (move_pages query)."""
    cap = max(1, (length + stride - 1) // stride)
    out = (C.c_int * cap)()
    n = C.c_uint64()
    _check(lib.lzckpt_numa_page_nodes(address, length, stride, out, cap, C.byref(n)))
    return list(out[:n.value])


def numa_prefer_range(address: int, length: int, node: int) -> None:
    _check(lib.lzckpt_numa_prefer_range(address, length, node))


def device_count() -> int:
    n = C.c_int()
    rc = dev.lzk_device_count(C.byref(n))
    return n.value if rc == 0 else 0


def kernel_launches() -> int:
    return dev.lzk_kernel_launches()


FNV_BASIS = 0xCBF29CE484222325


def _dev_check(rc: int) -> None:
    if rc != 0:
        raise (InvalidArgument if rc == 1 else DeviceError)(dev.lzk_last_error().decode(errors="replace"))


def device_fnv64(ranges: Sequence[Tuple[int, int]], device: int = 0, seeds: Optional[Sequence[int]] = None,
                 max_ctas: int = 0) -> List[int]:
    """FNV-1a-64 of device byte ranges [(address, length), ...] computed on
    the GPU (lzk_fnv1a64_batch), bit-identical to fnv64() of the same bytes;
    `seeds` continues from given states instead of the FNV basis."""
    n = len(ranges)
    if n == 0:
        return []
    out = C.c_void_p()
    _dev_check(dev.lzk_host_alloc(8 * n, 1, C.byref(out)))
    s = C.c_void_p()
    try:
        _dev_check(dev.lzk_stream_create(device, 0, C.byref(s)))
        arr = (N.HashDescC * n)()
        for i, (ptr, ln) in enumerate(ranges):
            arr[i] = N.HashDescC(ptr, ln, FNV_BASIS if seeds is None else seeds[i], out.value + 8 * i)
        _dev_check(dev.lzk_fnv1a64_batch(s, arr, n, max_ctas))
        _dev_check(dev.lzk_stream_sync(s))
        return list((C.c_uint64 * n).from_address(out.value))
    finally:
        if s.value:
            dev.lzk_stream_destroy(s)
        dev.lzk_host_free(out)


@dataclasses.dataclass
class BuiltWorkload:
    tree: StateTree
    model: ModelSpec
    topo: ParallelTopology
    rank: RankCoord
    step: int
    bytes: int


def build_workload(spec_path: str, device: int = 0) -> BuiltWorkload:
    """Materialize a workload spec (workloads.py) in HBM through the engine's
    own generator (GPU splitmix64 / host mt19937_64)."""
    t = C.c_void_p()
    m, tp = N.ModelSpecC(), N.Topology()
    rank = (C.c_uint32 * 3)()
    step, nbytes = C.c_uint64(), C.c_uint64()
    _check(lib.lzckpt_workload_build(os.fspath(spec_path).encode(), device, C.byref(t), C.byref(m), C.byref(tp),
                                     rank, C.byref(step), C.byref(nbytes)))
    return BuiltWorkload(StateTree(_handle=t),
                         ModelSpec("", m.param_count, m.layer_count, m.hidden_dim, m.bytes_per_param_model,
                                   m.bytes_per_param_optimizer),
                         ParallelTopology(tp.dp, tp.pp, tp.tp, tp.gpus_per_node, tp.node_count),
                         RankCoord(rank[0], rank[1], rank[2]), step.value, nbytes.value)
