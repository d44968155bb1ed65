"""Loader for the in-tree native libraries (built by ``__graft_entry__.build``).

There is no Python or CPU fallback for the snapshot path: if the shared
library is missing this module raises ImportError, and device calls on a box
without a GPU raise ``DeviceError`` from the native layer.
"""
from __future__ import annotations

import ctypes as C
import os

LIB_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib")
ENGINE_SO = os.path.join(LIB_DIR, "liblzckpt_b200.so")
DEVICE_SO = os.path.join(LIB_DIR, "liblzk_cuda.so")

if not os.path.exists(ENGINE_SO):
    raise ImportError(
        f"lzckpt native engine not built: {ENGINE_SO} is missing "
        "(run `python -c 'import __graft_entry__ as g; g.build()'`)")

# liblzckpt_b200.so finds liblzk_cuda.so through its $ORIGIN rpath.
dev = C.CDLL(DEVICE_SO, mode=C.RTLD_GLOBAL)
lib = C.CDLL(ENGINE_SO, mode=C.RTLD_GLOBAL)

u8p = C.POINTER(C.c_uint8)
u32, u64, i32, i64, f64 = C.c_uint32, C.c_uint64, C.c_int, C.c_int64, C.c_double
vp, cp = C.c_void_p, C.c_char_p


class Topology(C.Structure):
    _fields_ = [("dp", u32), ("pp", u32), ("tp", u32), ("gpus_per_node", u32), ("node_count", u32)]


class ModelSpecC(C.Structure):
    _fields_ = [("param_count", u64), ("layer_count", u32), ("hidden_dim", u32),
                ("bytes_per_param_model", u32), ("bytes_per_param_optimizer", u32)]


class ShardC(C.Structure):
    _fields_ = [("shard_id", u64), ("kind", u32), ("first_layer", u32), ("layer_count", u32),
                ("partition", u32), ("size_bytes", u64), ("owner_dp", u32), ("owner_pp", u32),
                ("owner_tp", u32), ("filename", C.c_char * 64)]


class HeaderEntryC(C.Structure):
    _fields_ = [("key", vp), ("key_len", u32), ("offset", u64), ("length", u64), ("checksum", u64)]


class EngineConfigC(C.Structure):
    _fields_ = [("checkpoint_root", cp), ("host_buffer_bytes", u64), ("copy_bandwidth_Bps", f64),
                ("chunk_quantum", u64), ("storage_bandwidth_Bps", f64), ("fsync_on_finalize", i32),
                ("flush_threads", u32), ("large_leaf_threshold", u64), ("reserve_timeout_ms", i64),
                ("device", i32), ("ce_threshold", u64), ("kernel_ctas", u32), ("group_bytes", u64),
                ("force_kernel", i32), ("force_copy_engine", i32), ("hugepages", i32),
                ("flush_discard", i32), ("stream_segment_bytes", u64), ("flush_hash_only", i32),
                ("relay_serve_socket", cp), ("relay_staging_bytes", u64), ("relay_ctas", u32),
                ("relay_peer_socket", cp), ("relay_share", f64), ("relay_min_entry", u64),
                ("relay_kernel_route", i32), ("flush_max_writers", u32),
                ("flush_write_piece", u64)]


class IpcHandleC(C.Structure):
    _fields_ = [("bytes", C.c_ubyte * 64)]


class CountersC(C.Structure):
    _fields_ = [("captures", u64), ("bytes_captured", u64), ("capture_seconds", f64),
                ("barrier_seconds", f64), ("last_capture_seconds", f64), ("last_barrier_seconds", f64)]


class SnapshotStatsC(C.Structure):
    _fields_ = [("kernel_launches", u64), ("kernel_bytes", u64), ("ce_copies", u64),
                ("ce_bytes", u64), ("blob_bytes", u64), ("groups", u64)]


class CopyDescC(C.Structure):
    _fields_ = [("src", u64), ("dst", u64), ("len", u64)]


class HashDescC(C.Structure):
    _fields_ = [("src", u64), ("len", u64), ("seed", u64), ("out", u64)]


P = C.POINTER

# (name, restype, argtypes) of every exported C-ABI symbol; tests check that
# each one declared in include/*.h is present and typed.
ENGINE_SYMBOLS = [
    ("lzckpt_last_error", cp, []),
    ("lzckpt_build_info", cp, []),
    ("lzckpt_fnv1a64", u64, [vp, u64]),
    ("lzckpt_fnv1a64_update", u64, [u64, vp, u64]),
    ("lzckpt_ring_create", i32, [u64, P(vp)]),
    ("lzckpt_ring_destroy", None, [vp]),
    ("lzckpt_ring_try_reserve", i32, [vp, u64, u64, P(u64), P(u64)]),
    ("lzckpt_ring_mark_filled", i32, [vp, u64]),
    ("lzckpt_ring_begin_flush", i32, [vp, u64]),
    ("lzckpt_ring_release", i32, [vp, u64]),
    ("lzckpt_ring_live_bytes", u64, [vp]),
    ("lzckpt_ring_live_segments", u64, [vp]),
    ("lzckpt_ring_released_bytes", u64, [vp]),
    ("lzckpt_ring_segment", i32, [vp, u64, P(u64), P(u64), P(i32)]),
    ("lzckpt_header_serialized_size", u64, [P(HeaderEntryC), u32]),
    ("lzckpt_header_serialize", i32, [P(HeaderEntryC), u32, u32, vp, u64, P(u64)]),
    ("lzckpt_header_parse", i32, [vp, u64, P(vp)]),
    ("lzckpt_file_read_header", i32, [cp, P(vp)]),
    ("lzckpt_header_destroy", None, [vp]),
    ("lzckpt_header_count", u32, [vp]),
    ("lzckpt_header_version", u32, [vp]),
    ("lzckpt_header_size", u64, [vp]),
    ("lzckpt_header_payload_end", u64, [vp]),
    ("lzckpt_header_entry_at", i32, [vp, u32, P(HeaderEntryC)]),
    ("lzckpt_file_validate", i32, [cp, vp, cp, u64, P(u32)]),
    ("lzckpt_plan_shards", i32, [P(Topology), P(ModelSpecC), u32, P(ShardC), u32, P(u32)]),
    ("lzckpt_region_create", i32, [i32, u64, P(vp)]),
    ("lzckpt_region_from_host", i32, [i32, vp, u64, P(vp)]),
    ("lzckpt_region_wrap", i32, [i32, vp, u64, P(vp)]),
    ("lzckpt_region_release", None, [vp]),
    ("lzckpt_region_size", u64, [vp]),
    ("lzckpt_region_version", u64, [vp]),
    ("lzckpt_region_device_ptr", vp, [vp]),
    ("lzckpt_region_device", i32, [vp]),
    ("lzckpt_region_read", i32, [vp, u64, vp, u64]),
    ("lzckpt_region_write", i32, [vp, u64, vp, u64]),
    ("lzckpt_region_mutate", i32, [vp, vp, u64]),
    ("lzckpt_region_bump_version", i32, [vp]),
    ("lzckpt_tree_create", i32, [P(vp)]),
    ("lzckpt_tree_destroy", None, [vp]),
    ("lzckpt_tree_set_region", i32, [vp, cp, vp]),
    ("lzckpt_tree_set_blob", i32, [vp, cp, vp, u64]),
    ("lzckpt_tree_leaf_count", u64, [vp]),
    ("lzckpt_tree_total_bytes", u64, [vp]),
    ("lzckpt_tree_leaf", i32, [vp, u64, cp, u64, P(i32), P(u64)]),
    ("lzckpt_tree_region_at", i32, [vp, cp, P(vp)]),
    ("lzckpt_tree_blob_at", i32, [vp, cp, vp, u64, P(u64)]),
    ("lzckpt_manifest_open", i32, [cp, P(vp)]),
    ("lzckpt_manifest_destroy", None, [vp]),
    ("lzckpt_manifest_commit_step", i32, [vp, u64, P(cp), P(u64), P(u64), u32]),
    ("lzckpt_manifest_is_committed", i32, [vp, u64]),
    ("lzckpt_manifest_latest", i32, [vp, P(i32), P(u64)]),
    ("lzckpt_engine_config_defaults", None, [P(EngineConfigC)]),
    ("lzckpt_engine_create", i32, [P(EngineConfigC), P(Topology), u32, u32, u32, P(vp)]),
    ("lzckpt_engine_destroy", None, [vp]),
    ("lzckpt_engine_capture", i32, [vp, P(ModelSpecC), vp, u64, P(vp)]),
    ("lzckpt_engine_capture_on_stream", i32, [vp, P(ModelSpecC), vp, u64, vp, P(vp)]),
    ("lzckpt_engine_update_barrier", i32, [vp, vp]),
    ("lzckpt_engine_update_barrier_on_stream", i32, [vp, vp, vp]),
    ("lzckpt_engine_wait_persisted", i32, [vp, vp]),
    ("lzckpt_engine_drain", i32, [vp]),
    ("lzckpt_engine_restore", i32, [vp, vp, u64, P(vp)]),
    ("lzckpt_engine_restore_into", i32, [vp, vp, u64, vp]),
    ("lzckpt_engine_counters", i32, [vp, P(CountersC)]),
    ("lzckpt_engine_snapshot_stats", i32, [vp, P(SnapshotStatsC)]),
    ("lzckpt_engine_flush_stats", i32, [vp, P(u64), P(u64)]),
    ("lzckpt_engine_snapshot_stream", vp, [vp]),
    ("lzckpt_engine_set_copy_variant", i32, [vp, u64, i32, i32, u32, u64]),
    ("lzckpt_engine_capture_file", i32, [vp, cp, vp, u64, P(vp)]),
    ("lzckpt_engine_capture_file_on_stream", i32, [vp, cp, vp, u64, vp, P(vp)]),
    ("lzckpt_engine_commit", i32, [vp, P(ModelSpecC), vp, vp, P(i32), cp, u64]),
    ("lzckpt_file_digest", i32, [cp, i32, P(u64), P(u64)]),
    ("lzckpt_trim_caches", None, []),
    ("lzckpt_numa_node_count", i32, []),
    ("lzckpt_numa_prefer_range", i32, [vp, u64, i32]),
    ("lzckpt_numa_page_nodes", i32, [vp, u64, u64, P(i32), u64, P(u64)]),
    ("lzckpt_engine_numa_node", i32, [vp]),
    ("lzckpt_engine_relay_stats", i32, [vp, P(u64), P(u64), P(u64)]),
    ("lzckpt_engine_set_relay", i32, [vp, cp, f64]),
    ("lzckpt_engine_prepare", i32, [vp, P(ModelSpecC), vp, cp, u64, P(u64)]),
    ("lzckpt_engine_ticket_header", i32, [vp, vp, u32, P(vp)]),
    ("lzckpt_engine_restore_file", i32, [vp, cp, vp, P(vp)]),
    ("lzckpt_ticket_release", None, [vp]),
    ("lzckpt_ticket_id", u64, [vp]),
    ("lzckpt_ticket_step", u64, [vp]),
    ("lzckpt_ticket_status", i32, [vp]),
    ("lzckpt_ticket_torn", i32, [vp]),
    ("lzckpt_ticket_payload_bytes", u64, [vp]),
    ("lzckpt_ticket_file_count", u32, [vp]),
    ("lzckpt_ticket_file", i32, [vp, u32, cp, u64]),
    ("lzckpt_ticket_failure_reason", i32, [vp, cp, u64]),
    ("lzckpt_engine_ticket_device_ms", f64, [vp, vp]),
    ("lzckpt_workload_build", i32, [cp, i32, P(vp), P(ModelSpecC), P(Topology), P(u32), P(u64), P(u64)]),
]

DEVICE_SYMBOLS = [
    ("lzk_last_error", cp, []),
    ("lzk_device_count", i32, [P(i32)]),
    ("lzk_set_device", i32, [i32]),
    ("lzk_get_device", i32, [P(i32)]),
    ("lzk_kernel_launches", u64, []),
    ("lzk_dev_alloc", i32, [i32, u64, P(vp)]),
    ("lzk_dev_free", i32, [i32, vp]),
    ("lzk_dev_memset", i32, [i32, vp, i32, u64]),
    ("lzk_memcpy_h2d", i32, [i32, vp, vp, u64]),
    ("lzk_memcpy_d2h", i32, [i32, vp, vp, u64]),
    ("lzk_memcpy_d2d", i32, [i32, vp, vp, u64]),
    ("lzk_host_alloc", i32, [u64, i32, P(vp)]),
    ("lzk_host_alloc_numa", i32, [u64, i32, i32, P(vp)]),
    ("lzk_device_numa_node", i32, [i32, P(i32)]),
    ("lzk_ipc_export_mem", i32, [i32, vp, P(IpcHandleC), P(u64)]),
    ("lzk_ipc_open_mem", i32, [i32, P(IpcHandleC), P(vp)]),
    ("lzk_ipc_close_all", i32, []),
    ("lzk_ipc_event_create", i32, [i32, P(vp), P(IpcHandleC)]),
    ("lzk_ipc_event_open", i32, [i32, P(IpcHandleC), P(vp)]),
    ("lzk_host_free", i32, [vp]),
    ("lzk_host_register", i32, [vp, u64]),
    ("lzk_host_unregister", i32, [vp]),
    ("lzk_stream_create", i32, [i32, i32, P(vp)]),
    ("lzk_stream_wrap", i32, [i32, vp, P(vp)]),
    ("lzk_stream_destroy", i32, [vp]),
    ("lzk_stream_sync", i32, [vp]),
    ("lzk_stream_handle", vp, [vp]),
    ("lzk_stream_device", i32, [vp]),
    ("lzk_event_create", i32, [i32, i32, P(vp)]),
    ("lzk_event_destroy", i32, [vp]),
    ("lzk_event_record", i32, [vp, vp]),
    ("lzk_event_query", i32, [vp]),
    ("lzk_event_sync", i32, [vp]),
    ("lzk_event_elapsed_ms", i32, [vp, vp, P(C.c_float)]),
    ("lzk_stream_wait_event", i32, [vp, vp]),
    ("lzk_raw_stream_wait_event", i32, [vp, vp]),
    ("lzk_event_record_raw", i32, [vp, vp]),
    ("lzk_stream_wait_raw", i32, [vp, vp]),
    ("lzk_gather_d2h", i32, [vp, P(CopyDescC), u32, u32]),
    ("lzk_ce_copy_d2h", i32, [vp, P(CopyDescC), u32]),
    ("lzk_scatter_h2d", i32, [vp, P(CopyDescC), u32, u32]),
    ("lzk_ce_copy_h2d", i32, [vp, P(CopyDescC), u32]),
    ("lzk_ce_copy_d2d", i32, [vp, P(CopyDescC), u32]),
    ("lzk_gather_d2d", i32, [vp, P(CopyDescC), u32, u32]),
    ("lzk_fnv1a64_batch", i32, [vp, P(HashDescC), u32, u32]),
    ("lzk_fnv1a64_continue", i32, [vp, P(HashDescC), u32, u32]),
    ("lzk_fill_splitmix", i32, [vp, vp, u64, u64, u64]),
    ("lzk_busy_compute", i32, [vp, vp, u64, u32, u32]),
    ("lzk_range_push", None, [cp]),
    ("lzk_range_pop", None, []),
]


def _bind(handle, table):
    for name, res, args in table:
        fn = getattr(handle, name)  # AttributeError = missing export: fail loudly
        fn.restype = res
        fn.argtypes = args


_bind(lib, ENGINE_SYMBOLS)
_bind(dev, DEVICE_SYMBOLS)
