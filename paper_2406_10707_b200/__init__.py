"""B200-native lazy asynchronous snapshot engine (DataStates-LLM path, arxiv 2406.10707).

The product is the native pair under ``lib/``: ``liblzk_cuda.so`` (sm_100a
kernels + the include/lzk_cuda.h C ABI) and ``liblzckpt_b200.so`` (the C++
engine + include/lzckpt_c.h). This package is the Python mirror of the
reference ``lzckpt`` API over that C ABI.
"""
from .lzckpt import *  # noqa: F401,F403
from .lzckpt import (CaptureTicket, CheckpointFileHeader, CheckpointPlan, DeviceRegion, Engine,  # noqa: F401
                     EngineConfig, HeaderEntry, ManifestStore, ModelSpec, ParallelTopology, RankCoord,
                     RingCore, StateTree, committed_record, device_count, device_fnv64, fnv64, kernel_launches,
                     parse_header, plan_checkpoint, read_entry, read_header, serialize_header,
                     validate_entries)
