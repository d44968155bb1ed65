"""DeepSpeed-style checkpoint engine over the B200 lazy snapshot path
("framework glue").

DataStates-LLM ships as a DeepSpeed checkpoint engine whose primitives are
DeepSpeed's (``create``, ``makedirs``, ``save``, ``load``, ``commit``) plus one
extra blocking ``wait`` for pending snapshot captures (PAPER.md §"Architecture",
lines 612-619). This class offers that surface on top of ``Engine.capture_file``:

* ``save(state_dict, path)`` walks the Python object, registers every CUDA
  tensor zero-copy as a device region (CPU tensors and other objects travel
  as host blobs / a pickled skeleton), and returns after the capture is queued;
  the D2H snapshot, per-entry checksums and the file write run behind training.
* ``wait(stream=None)`` is the lazy fence: call it before the optimizer mutates
  the saved tensors. With a CUDA stream it is a device-side wait (the host
  does not block).
* ``commit(tag)`` blocks until every file of the tag is durable.
* ``load(path, map_location=None)`` validates the file and DMAs tensors
  straight into freshly allocated torch tensors.

Files are LZCKPT01 shard files (the reference format), one per ``save`` call.
"""
from __future__ import annotations

import io
import os
import pickle
import struct
import tempfile
from typing import Any, Dict, List, Optional

from . import lzckpt as L

SKELETON = "__skeleton__"


def _component(i: int, key: Any) -> str:
    """Path component for the i-th child: unique (index prefix) and free of '/'."""
    text = str(key).replace("/", "∕") if isinstance(key, (str, int)) else type(key).__name__
    return f"{i}:{text}" if text else str(i)


class DataStatesCheckpointEngine:
    def __init__(self, config_params: Optional[dict] = None, host_cache_bytes: Optional[int] = None,
                 device: Optional[int] = None, large_leaf_threshold: int = 1 << 20):
        import torch
        cfg = dict(config_params or {})
        cfg = cfg.get("datastates_ckpt", cfg)
        host = host_cache_bytes or int(cfg.get("host_cache_size", 16 << 30))
        dev = torch.cuda.current_device() if device is None else device
        self.device = dev
        # Files larger than the host cache stream through it (backpressure).
        self._engine = L.Engine(L.EngineConfig(checkpoint_root=tempfile.gettempdir(), host_buffer_bytes=host,
                                               large_leaf_threshold=large_leaf_threshold, device=dev,
                                               fsync_on_finalize=bool(cfg.get("fsync", True)),
                                               stream_segment_bytes=max(host // 4, 1 << 20)),
                                L.ParallelTopology(1, 1, 1, 1, 1), L.RankCoord())
        self._pending: List[L.CaptureTicket] = []
        self._keep: List[L.StateTree] = []  # tensors stay referenced until persisted
        self._step = 0
        self.tag = None

    # -- DeepSpeed CheckpointEngine primitives ---------------------------------
    def create(self, tag) -> None:
        self.tag = tag

    def makedirs(self, path, exist_ok: bool = False) -> None:
        os.makedirs(path, exist_ok=exist_ok)

    def save(self, state_dict: Any, path: str, stream=None) -> None:
        """Queues the snapshot and returns. It is ordered on the device after
        the work already queued on `stream` (default: the current torch stream),
        so a save right after an un-synchronised optimizer.step() reads the
        updated tensors, never half-written ones."""
        import torch
        tree = L.StateTree()
        skeleton = self._flatten(state_dict, "s", tree)
        tree.set_blob(SKELETON, pickle.dumps(skeleton, protocol=pickle.HIGHEST_PROTOCOL))
        self._step += 1
        producer = torch.cuda.current_stream(self.device) if stream is None else stream
        self._pending.append(self._engine.capture_file(path, tree, self._step, producer_stream=producer))
        self._keep.append(tree)

    def wait(self, stream=None) -> None:
        """Block (or make `stream` wait) until every pending snapshot is in host
        memory; after this the saved tensors may be mutated."""
        for t in self._pending:
            if stream is None:
                self._engine.update_barrier(t)
            else:
                self._engine.update_barrier_on_stream(t, getattr(stream, "cuda_stream", stream))

    def commit(self, tag=None) -> bool:
        try:
            for t in self._pending:
                self._engine.wait_persisted(t)
        finally:
            self._pending.clear()
            self._keep.clear()
        return True

    def load(self, path: str, map_location=None) -> Any:
        import torch
        skeleton = pickle.loads(_read_blob(path, SKELETON))
        specs: Dict[str, tuple] = {}
        _collect_specs(skeleton, specs)
        target = None
        if map_location is not None:
            target = torch.device(map_location) if not callable(map_location) else None
        into = L.StateTree()
        tensors: Dict[str, Any] = {}
        for p, (dtype, shape, device, is_region) in specs.items():
            dev = target or torch.device(device)
            if is_region and dev.type == "cuda":
                t = torch.empty(shape, dtype=getattr(torch, dtype), device=dev)
                tensors[p] = t
                into.set_region(p, L.DeviceRegion.wrap(t))
        back = self._engine.restore_file(path, into)
        for p, (dtype, shape, device, is_region) in specs.items():
            if p in tensors:
                continue
            raw = back.region_at(p).clone_bytes() if is_region else back.blob_at(p)
            t = torch.frombuffer(bytearray(raw), dtype=torch.uint8) if raw else torch.empty(0, dtype=torch.uint8)
            t = t.view(getattr(torch, dtype)).reshape(shape)
            dev = target or torch.device(device)
            tensors[p] = t.to(dev) if dev.type != "cpu" else t
        return _rebuild(skeleton, tensors)

    def close(self) -> None:
        self.commit()
        self._engine.close()

    # -- object walk -------------------------------------------------------------
    # skeleton nodes: ("t", path, dtype, shape, device, on_gpu) tensor leaf,
    # ("d", type, [(key, node)...]) mapping, ("l", type, [node...]) sequence,
    # ("o", obj) anything else (pickled as is)
    def _flatten(self, obj: Any, path: str, tree: L.StateTree) -> Any:
        import torch
        if isinstance(obj, torch.Tensor):
            t = obj.detach()
            dtype = str(t.dtype).replace("torch.", "")
            if t.is_cuda:
                if not t.is_contiguous():
                    t = t.contiguous()  # the snapshot holds this copy until committed
                tree.set_region(path, L.DeviceRegion.wrap(t.reshape(-1), device=t.device.index))
                return ("t", path, dtype, tuple(obj.shape), str(obj.device), True)
            raw = t.contiguous().reshape(-1).view(torch.uint8).numpy().tobytes() if t.numel() else b""
            tree.set_blob(path, raw)
            return ("t", path, dtype, tuple(obj.shape), "cpu", False)
        if isinstance(obj, dict):
            return ("d", type(obj), [(k, self._flatten(v, f"{path}/{_component(i, k)}", tree))
                                     for i, (k, v) in enumerate(obj.items())])
        if isinstance(obj, (list, tuple)):
            return ("l", type(obj), [self._flatten(v, f"{path}/{i}", tree) for i, v in enumerate(obj)])
        return ("o", obj)


def _collect_specs(node: Any, out: Dict[str, tuple]) -> None:
    tag = node[0]
    if tag == "t":
        out[node[1]] = node[2:]
    elif tag == "d":
        for _, child in node[2]:
            _collect_specs(child, out)
    elif tag == "l":
        for child in node[2]:
            _collect_specs(child, out)


def _rebuild(node: Any, tensors: Dict[str, Any]) -> Any:
    tag = node[0]
    if tag == "t":
        return tensors[node[1]]
    if tag == "o":
        return node[1]
    if tag == "d":
        d = node[1]()
        for k, child in node[2]:
            d[k] = _rebuild(child, tensors)
        return d
    items = [_rebuild(child, tensors) for child in node[2]]
    return items if node[1] is list else node[1](items)


def _read_blob(path: str, key: str) -> bytes:
    """A blob leaf straight from the file: a large blob is its own entry, a
    small one rides inside __meta__ (u32 n; n x {u32 len, path, u8 flags,
    u64 size, [bytes]}, reference state_tree.cpp:195-210)."""
    h = L.read_header(path)
    if h.find(key) is not None:
        return L.read_entry(path, h, key)
    meta = io.BytesIO(L.read_entry(path, h, "__meta__"))
    (n,) = struct.unpack("<I", meta.read(4))
    for _ in range(n):
        (ln,) = struct.unpack("<I", meta.read(4))
        p = meta.read(ln).decode()
        flags, size = struct.unpack("<BQ", meta.read(9))
        data = meta.read(size) if flags & 2 else None
        if p == key and data is not None:
            return data
    raise L.FormatError(f"{path}: no blob '{key}'")
