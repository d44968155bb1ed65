/*
 * lzk_cuda.h — thin C ABI between the lzckpt host engine (C++) and the
 * B200 device layer (sm_100a CUDA). No CUDA or torch types cross it: device
 * and host memory are plain pointers, streams/events are opaque handles.
 *
 * Conventions
 *   - every call returns int status (LZK_OK = 0); on failure a thread-local
 *     message is available from lzk_last_error();
 *   - no C++ exception crosses the ABI;
 *   - descriptor arrays are borrowed for the duration of the call only: the
 *     callee stages them into its own pinned/device memory before returning;
 *   - calls that take a `device` argument make it current on the calling
 *     thread; stream-taking calls use the stream's device.
 *
 * What each entry point replaces in the reference (paths relative to
 * /root/reference/proj/core):
 *   lzk_gather_d2h / lzk_ce_copy_d2h
 *       TransferEngine::run_task's chunked memcpy loop and
 *       DeviceRegion::read_chunk (src/transfer_engine.cpp:117-160, :25-31);
 *       also the per-leaf DeviceRegion::clone_bytes of Engine::capture's
 *       inline leaves (src/engine.cpp:138-143, src/transfer_engine.cpp:33-36).
 *   lzk_scatter_h2d / lzk_ce_copy_h2d
 *       Engine::restore's "new DeviceRegion from host bytes"
 *       (src/engine.cpp:371-372).
 *   lzk_event_* / lzk_stream_wait_event
 *       TransferEngine::wait_pending's condition-variable wait
 *       (src/transfer_engine.cpp:162-174) — the lazy fence.
 *   lzk_host_alloc
 *       HostBufferPool's std::vector storage (src/buffer_pool.cpp:10):
 *       pinned + mapped so the copy engine and SM stores reach it directly.
 *   lzk_fnv1a64_batch
 *       Fnv64 / fnv64 (include/lzckpt/checksum.hpp:12-43) as used for the
 *       per-entry checksums of FlushPipeline::write_chunk/finalize
 *       (src/flush_pipeline.cpp:194-263) and the restore check in
 *       validate_entries/read_entry (src/format.cpp:173-214).
 *   lzk_dev_alloc / lzk_memcpy_* / lzk_dev_memset
 *       DeviceRegion's host std::vector (include/lzckpt/transfer_engine.hpp:24-43).
 */
#ifndef LZK_CUDA_H_
#define LZK_CUDA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LZK_OK 0
#define LZK_ERR_INVALID 1   /* bad argument */
#define LZK_ERR_CUDA 2      /* CUDA runtime failure (message has details) */
#define LZK_ERR_NODEV 3     /* no CUDA device visible */
#define LZK_ERR_NOMEM 4     /* host or device allocation failed */
#define LZK_PENDING 5       /* lzk_event_query: work not finished yet */

/* One copy: `len` bytes from `src` to `dst`. For D2H, src is a device
 * address and dst a pinned, mapped host address; for H2D the reverse.
 * Both may have any byte alignment. */
typedef struct lzk_copy_desc {
  uint64_t src;
  uint64_t dst;
  uint64_t len;
} lzk_copy_desc;

/* One checksum: FNV-1a-64 of `len` bytes at device address `src` (any
 * alignment), continuing from state `seed` (LZK_FNV_BASIS for a fresh
 * digest). The 8-byte result is stored at `out`: device memory or pinned,
 * mapped host memory. */
typedef struct lzk_hash_desc {
  uint64_t src;
  uint64_t len;
  uint64_t seed;
  uint64_t out;
} lzk_hash_desc;
#define LZK_FNV_BASIS 0xcbf29ce484222325ull

typedef struct lzk_stream lzk_stream;
typedef struct lzk_event lzk_event;

const char* lzk_last_error(void);
int lzk_device_count(int* count);
int lzk_set_device(int device);
int lzk_get_device(int* device);
/* Kernel launches this process made through lzk_* (gather, scatter, fill,
 * hash); used by bench.py to report gpu_launches. */
uint64_t lzk_kernel_launches(void);

/* ---- device memory ---------------------------------------------------- */
int lzk_dev_alloc(int device, uint64_t bytes, void** ptr);
int lzk_dev_free(int device, void* ptr);
int lzk_dev_memset(int device, void* ptr, int value, uint64_t bytes); /* synchronous */
/* Synchronous copies on an internal per-device stream (never the legacy
 * default stream, so they do not serialize against snapshot streams). */
int lzk_memcpy_h2d(int device, void* dst, const void* src, uint64_t bytes);
int lzk_memcpy_d2h(int device, void* dst, const void* src, uint64_t bytes);
int lzk_memcpy_d2d(int device, void* dst, const void* src, uint64_t bytes);

/* ---- pinned host memory ----------------------------------------------- */
#define LZK_HOST_MAPPED 0x1    /* device-visible alias (UVA: same address) */
#define LZK_HOST_HUGEPAGE 0x2  /* mmap + MADV_HUGEPAGE + parallel first touch + register */
int lzk_host_alloc(uint64_t bytes, int flags, void** ptr);
/* Same, with the pages placed on `numa_node` (MPOL_PREFERRED set before the
 * first touch, which that node's CPUs perform); -1 = no placement. */
int lzk_host_alloc_numa(uint64_t bytes, int flags, int numa_node, void** ptr);
/* NUMA node of the GPU's PCI function (/sys/bus/pci/devices/<bdf>/numa_node);
 * -1 when the host does not report one (single-node machines). */
int lzk_device_numa_node(int device, int* node);
int lzk_host_free(void* ptr);
/* Pins an existing host range (e.g. a numpy buffer) for direct DMA. */
int lzk_host_register(void* ptr, uint64_t bytes);
int lzk_host_unregister(void* ptr);

/* ---- streams and events ------------------------------------------------ */
/* priority: <0 = the greatest priority; 0 and >0 = the least, which on
 * current GPUs is also the default (CUDA has nothing below an ordinary
 * stream). */
int lzk_stream_create(int device, int priority, lzk_stream** s);
/* Wraps a foreign cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream)
 * without taking ownership. */
int lzk_stream_wrap(int device, void* cuda_stream, lzk_stream** s);
int lzk_stream_destroy(lzk_stream* s);
int lzk_stream_sync(lzk_stream* s);
void* lzk_stream_handle(lzk_stream* s);
int lzk_stream_device(lzk_stream* s);

/* blocking_sync != 0: lzk_event_sync yields the CPU instead of spinning. */
int lzk_event_create(int device, int blocking_sync, lzk_event** e);
int lzk_event_destroy(lzk_event* e);
int lzk_event_record(lzk_event* e, lzk_stream* s);
int lzk_event_query(lzk_event* e); /* LZK_OK done, LZK_PENDING not yet */
int lzk_event_sync(lzk_event* e);
int lzk_event_elapsed_ms(lzk_event* start, lzk_event* end, float* ms);
/* Device-side fence: work queued on `s` after this call waits for `e`. */
int lzk_stream_wait_event(lzk_stream* s, lzk_event* e);
/* Records `e` on a raw cudaStream_t owned by the caller (NULL = the legacy
 * default stream): how capture() marks "everything the trainer has queued so
 * far" on the producer stream before the snapshot stream waits for it. */
int lzk_event_record_raw(lzk_event* e, void* cuda_stream);
/* `s` waits for the work queued so far on a raw producer stream (NULL = the
 * legacy default stream). */
int lzk_stream_wait_raw(lzk_stream* s, void* producer_stream);
/* Same, for a raw cudaStream_t handle owned by the caller. */
int lzk_raw_stream_wait_event(void* cuda_stream, lzk_event* e);

/* ---- CUDA IPC (uplink relay between the ranks of one node) -------------- */
/* 64 opaque bytes: a cudaIpcMemHandle_t or cudaIpcEventHandle_t. */
typedef struct lzk_ipc_handle {
  unsigned char bytes[64];
} lzk_ipc_handle;
/* IPC handle of the allocation holding `dev_ptr` and dev_ptr's offset in it
 * (works for torch tensors inside larger allocator blocks). */
int lzk_ipc_export_mem(int device, const void* dev_ptr, lzk_ipc_handle* handle, uint64_t* offset);
/* Maps a peer process's allocation into this process (with peer access);
 * cached: each handle opens once per process and device. */
int lzk_ipc_open_mem(int device, const lzk_ipc_handle* handle, void** base);
int lzk_ipc_close_all(void);
/* Interprocess event (no timing) and its handle; the peer opens it with
 * lzk_ipc_event_open and can record/wait/sync it like any lzk_event. */
int lzk_ipc_event_create(int device, lzk_event** e, lzk_ipc_handle* handle);
int lzk_ipc_event_open(int device, const lzk_ipc_handle* handle, lzk_event** e);

/* ---- the snapshot copies ----------------------------------------------- */
/* Multi-tensor gather D2H on SMs: one launch copies all n descriptors into
 * mapped pinned host memory with coalesced 128-bit loads and 16-byte aligned
 * stores (byte-granular destinations are realigned in registers).
 * max_ctas == 0 picks the default grid (a host-link-saturating handful). */
int lzk_gather_d2h(lzk_stream* s, const lzk_copy_desc* d, uint32_t n, uint32_t max_ctas);
/* Copy-engine variant: one DMA per descriptor on the stream (no SM use). */
int lzk_ce_copy_d2h(lzk_stream* s, const lzk_copy_desc* d, uint32_t n);
/* Restore direction: pinned host -> device. */
int lzk_scatter_h2d(lzk_stream* s, const lzk_copy_desc* d, uint32_t n, uint32_t max_ctas);
int lzk_ce_copy_h2d(lzk_stream* s, const lzk_copy_desc* d, uint32_t n);
/* Device-to-device copy-engine variant (also peer memory opened through IPC:
 * the uplink relay pulls a peer's tensors over NVLink this way). */
int lzk_ce_copy_d2d(lzk_stream* s, const lzk_copy_desc* d, uint32_t n);
/* Device-to-device multi-tensor gather (same kernel, device destination). */
int lzk_gather_d2d(lzk_stream* s, const lzk_copy_desc* d, uint32_t n, uint32_t max_ctas);

/* ---- checksums ----------------------------------------------------------- */
/* Device FNV-1a-64 of n byte ranges in stream order, bit-identical to the
 * reference's byte-serial fold. A bit-sliced scan of the low-byte trajectory
 * lets the 32 lanes of a warp hash one range in parallel; ranges larger than
 * a fair share of the grid are split into segments hashed by many warps
 * (multi-pass). max_ctas bounds the CTAs (SMs) used; 0 = two per SM. */
int lzk_fnv1a64_batch(lzk_stream* s, const lzk_hash_desc* d, uint32_t n, uint32_t max_ctas);
/* Same, continuing running digests: each range's initial state is read from
 * its `out` address (seed ignored) and the new state written back there. */
int lzk_fnv1a64_continue(lzk_stream* s, const lzk_hash_desc* d, uint32_t n, uint32_t max_ctas);

/* ---- profiler ranges -------------------------------------------------------- */
/* NVTX ranges (nsys / ncu timelines): no-ops unless a profiler is attached.
 * The engine marks capture, the lazy fences, flush finalize, restore and
 * commit validation with them. */
void lzk_range_push(const char* name);
void lzk_range_pop(void);

/* ---- synthetic workload generation (bench/tests) ------------------------ */
/* Fills `bytes` of device memory with the splitmix64 counter stream of
 * (seed, leaf): word w = mix64((seed ^ leaf*0xD1B54A32D192ED03) + (w+1)*0x9E3779B97F4A7C15),
 * little-endian; a final partial word donates its leading bytes. */
int lzk_fill_splitmix(lzk_stream* s, void* dev, uint64_t bytes, uint64_t seed, uint64_t leaf);
/* Busy kernel standing in for forward/backward compute: `iters` dependent FMA
 * rounds on every element of `buf` (n floats) using `ctas` CTAs. */
int lzk_busy_compute(lzk_stream* s, float* buf, uint64_t n, uint32_t iters, uint32_t ctas);

#ifdef __cplusplus
}
#endif
#endif /* LZK_CUDA_H_ */
