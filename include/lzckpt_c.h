/*
 * lzckpt_c.h — C ABI of the lzckpt snapshot engine (liblzckpt_b200.so).
 *
 * The reference exposes only a C++ API (the headers under proj/core/include/lzckpt); this
 * is the flat binding an FFI host (ctypes, cgo, JNI) would use for the same
 * path. Each entry point wraps exactly one reference call:
 *
 *   lzckpt_region_*          DeviceRegion            transfer_engine.hpp:24-43
 *   lzckpt_tree_*            StateTree               state_tree.hpp:19-79
 *   lzckpt_plan_shards       plan_checkpoint         topology.hpp:97-98
 *   lzckpt_engine_create     Engine::Engine          engine.hpp:88
 *   lzckpt_engine_capture    Engine::capture         engine.hpp:97-98 / engine.cpp:96-231
 *   lzckpt_engine_capture_on_stream  Engine::capture, ordered after a trainer stream
 *   lzckpt_engine_update_barrier
 *                            Engine::update_barrier  engine.hpp:103 / engine.cpp:233-253
 *   lzckpt_engine_wait_persisted, _drain, _restore, _counters
 *                            engine.hpp:105-120 / engine.cpp:255-379
 *   lzckpt_ticket_*          CaptureTicket           engine.hpp:32-68
 *   lzckpt_manifest_*        ManifestStore           manifest.hpp:29-49
 *   lzckpt_ring_*            RingCore                ring_core.hpp:31-68
 *   lzckpt_header_*, lzckpt_file_*
 *                            format.hpp:51-72
 *   lzckpt_fnv1a64*          Fnv64 / fnv64           checksum.hpp:12-43
 *
 * B200 extensions: lzckpt_engine_update_barrier_on_stream (device-side lazy
 * fence), lzckpt_engine_restore_into (in-place restore), region wrapping of
 * foreign device memory, snapshot statistics.
 *
 * Errors: every int-returning call returns LZCKPT_OK or the code of the C++
 * exception class it caught (one code per class of errors.hpp);
 * lzckpt_last_error() holds the message (thread-local).
 * Handles returned through out-pointers are owned by the caller and freed
 * with the matching *_release / *_destroy call.
 */
#ifndef LZCKPT_C_H_
#define LZCKPT_C_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LZCKPT_OK 0
#define LZCKPT_E_ERROR 1
#define LZCKPT_E_CONFIG 2
#define LZCKPT_E_SIZE_EXCEEDS 3
#define LZCKPT_E_WAIT_TIMEOUT 4
#define LZCKPT_E_ILLEGAL_TRANSITION 5
#define LZCKPT_E_TORN 6
#define LZCKPT_E_DUPLICATE_PATH 7
#define LZCKPT_E_FORMAT 8
#define LZCKPT_E_BAD_MAGIC 9
#define LZCKPT_E_TRUNCATED 10
#define LZCKPT_E_CHECKSUM 11
#define LZCKPT_E_NOT_COMMITTED 12
#define LZCKPT_E_CORRUPT_MANIFEST 13
#define LZCKPT_E_IO 14
#define LZCKPT_E_DEVICE 15
#define LZCKPT_E_INVALID 16

const char* lzckpt_last_error(void);
const char* lzckpt_build_info(void);

/* ---- checksum ---------------------------------------------------------- */
uint64_t lzckpt_fnv1a64(const void* data, uint64_t len);
uint64_t lzckpt_fnv1a64_update(uint64_t state, const void* data, uint64_t len);

/* ---- ring allocator state machine (pure host logic) -------------------- */
typedef struct lzckpt_ring lzckpt_ring;
int lzckpt_ring_create(uint64_t capacity, lzckpt_ring** out);
void lzckpt_ring_destroy(lzckpt_ring* r);
/* *id == 0 when nothing fits right now (RingCore::try_reserve -> nullopt). */
int lzckpt_ring_try_reserve(lzckpt_ring* r, uint64_t size, uint64_t ticket, uint64_t* id,
                            uint64_t* offset);
int lzckpt_ring_mark_filled(lzckpt_ring* r, uint64_t id);
int lzckpt_ring_begin_flush(lzckpt_ring* r, uint64_t id);
int lzckpt_ring_release(lzckpt_ring* r, uint64_t id);
uint64_t lzckpt_ring_live_bytes(const lzckpt_ring* r);
uint64_t lzckpt_ring_live_segments(const lzckpt_ring* r);
uint64_t lzckpt_ring_released_bytes(const lzckpt_ring* r);
/* state: 0 Reserved, 1 Filled, 2 Flushing, 3 Free; IllegalTransition if unknown */
int lzckpt_ring_segment(const lzckpt_ring* r, uint64_t id, uint64_t* offset, uint64_t* length,
                        int* state);

/* ---- shard-file header codec -------------------------------------------- */
typedef struct lzckpt_header_entry {
  const char* key; /* not NUL-terminated necessarily: key_len bytes */
  uint32_t key_len;
  uint64_t offset;
  uint64_t length;
  uint64_t checksum;
} lzckpt_header_entry;
typedef struct lzckpt_header lzckpt_header;
uint64_t lzckpt_header_serialized_size(const lzckpt_header_entry* e, uint32_t n);
/* Writes the serialized header into out (cap bytes); *size = bytes needed. */
int lzckpt_header_serialize(const lzckpt_header_entry* e, uint32_t n, uint32_t version, void* out,
                            uint64_t cap, uint64_t* size);
int lzckpt_header_parse(const void* bytes, uint64_t n, lzckpt_header** out);
int lzckpt_file_read_header(const char* path, lzckpt_header** out);
void lzckpt_header_destroy(lzckpt_header* h);
uint32_t lzckpt_header_count(const lzckpt_header* h);
uint32_t lzckpt_header_version(const lzckpt_header* h);
uint64_t lzckpt_header_size(const lzckpt_header* h);
uint64_t lzckpt_header_payload_end(const lzckpt_header* h);
/* key pointer stays valid until lzckpt_header_destroy */
int lzckpt_header_entry_at(const lzckpt_header* h, uint32_t i, lzckpt_header_entry* out);
/* Recomputes entry checksums; *n_bad = mismatching entries, their keys are
 * written '\n'-separated into bad_keys (cap bytes). */
int lzckpt_file_validate(const char* path, const lzckpt_header* h, char* bad_keys, uint64_t cap,
                         uint32_t* n_bad);

/* ---- topology / plan ------------------------------------------------------ */
typedef struct lzckpt_topology {
  uint32_t dp, pp, tp, gpus_per_node, node_count;
} lzckpt_topology;
typedef struct lzckpt_model_spec {
  uint64_t param_count;
  uint32_t layer_count;
  uint32_t hidden_dim;
  uint32_t bytes_per_param_model;
  uint32_t bytes_per_param_optimizer;
} lzckpt_model_spec;
typedef struct lzckpt_shard {
  uint64_t shard_id;
  uint32_t kind; /* 0 LayerShard, 1 OptimizerShard */
  uint32_t first_layer;
  uint32_t layer_count;
  uint32_t partition;
  uint64_t size_bytes;
  uint32_t owner_dp, owner_pp, owner_tp;
  char filename[64];
} lzckpt_shard;
int lzckpt_plan_shards(const lzckpt_topology* topo, const lzckpt_model_spec* model,
                       uint32_t flat_rank, lzckpt_shard* out, uint32_t cap, uint32_t* n);

/* ---- device regions ------------------------------------------------------ */
typedef struct lzckpt_region lzckpt_region;
int lzckpt_region_create(int device, uint64_t size, lzckpt_region** out);
int lzckpt_region_from_host(int device, const void* bytes, uint64_t size, lzckpt_region** out);
/* non-owning view of foreign device memory (e.g. a torch tensor) */
int lzckpt_region_wrap(int device, void* device_ptr, uint64_t size, lzckpt_region** out);
void lzckpt_region_release(lzckpt_region* r);
uint64_t lzckpt_region_size(const lzckpt_region* r);
uint64_t lzckpt_region_version(const lzckpt_region* r);
void* lzckpt_region_device_ptr(const lzckpt_region* r);
int lzckpt_region_device(const lzckpt_region* r);
int lzckpt_region_read(const lzckpt_region* r, uint64_t offset, void* out, uint64_t n);
int lzckpt_region_write(lzckpt_region* r, uint64_t offset, const void* data, uint64_t n);
/* DeviceRegion::mutate with fn = "overwrite with data" (one version bump) */
int lzckpt_region_mutate(lzckpt_region* r, const void* data, uint64_t n);
int lzckpt_region_bump_version(lzckpt_region* r);

/* ---- state tree ------------------------------------------------------------ */
typedef struct lzckpt_tree lzckpt_tree;
int lzckpt_tree_create(lzckpt_tree** out);
void lzckpt_tree_destroy(lzckpt_tree* t);
int lzckpt_tree_set_region(lzckpt_tree* t, const char* path, const lzckpt_region* r);
int lzckpt_tree_set_blob(lzckpt_tree* t, const char* path, const void* bytes, uint64_t n);
uint64_t lzckpt_tree_leaf_count(const lzckpt_tree* t);
uint64_t lzckpt_tree_total_bytes(const lzckpt_tree* t);
/* i-th leaf in flatten() order; path written NUL-terminated into path (cap). */
int lzckpt_tree_leaf(const lzckpt_tree* t, uint64_t i, char* path, uint64_t cap, int* is_region,
                     uint64_t* size);
int lzckpt_tree_region_at(const lzckpt_tree* t, const char* path, lzckpt_region** out);
int lzckpt_tree_blob_at(const lzckpt_tree* t, const char* path, void* out, uint64_t cap,
                        uint64_t* size);

/* ---- manifest ---------------------------------------------------------------- */
typedef struct lzckpt_manifest lzckpt_manifest;
int lzckpt_manifest_open(const char* path, lzckpt_manifest** out);
void lzckpt_manifest_destroy(lzckpt_manifest* m);
int lzckpt_manifest_commit_step(lzckpt_manifest* m, uint64_t step, const char* const* paths,
                                const uint64_t* lengths, const uint64_t* digests, uint32_t n);
int lzckpt_manifest_is_committed(const lzckpt_manifest* m, uint64_t step);
/* returns 0 and *has = 0 when nothing is committed */
int lzckpt_manifest_latest(const lzckpt_manifest* m, int* has, uint64_t* step);

/* ---- engine -------------------------------------------------------------------- */
typedef struct lzckpt_engine_config {
  const char* checkpoint_root;
  uint64_t host_buffer_bytes;
  double copy_bandwidth_Bps;  /* <= 0: unpaced (device fast path) */
  uint64_t chunk_quantum;
  double storage_bandwidth_Bps;
  int fsync_on_finalize;
  uint32_t flush_threads;     /* 0 = auto */
  uint64_t large_leaf_threshold;
  int64_t reserve_timeout_ms;
  int device;                 /* -1 = current */
  uint64_t ce_threshold;      /* tensors >= this use the copy engines */
  uint32_t kernel_ctas;
  uint64_t group_bytes;
  int force_kernel;
  int force_copy_engine;
  int hugepages;
  int flush_discard;          /* host-memory tier only (no files) */
  uint64_t stream_segment_bytes; /* > 0: files stream through the pool in segments this large */
  int flush_hash_only;        /* verification tier: hash every entry, write nothing */
  /* uplink relay between the ranks of one node (EngineConfig::Relay) */
  const char* relay_serve_socket;   /* helper: serve relay requests here (NULL/"" = no) */
  uint64_t relay_staging_bytes;
  uint32_t relay_ctas;
  const char* relay_peer_socket;    /* owner: delegate to the helper listening here */
  double relay_share;               /* fraction of each shard file's payload (0 = off) */
  uint64_t relay_min_entry;
  int relay_kernel_route;           /* helper: 1 = SM gather kernel, 0 = copy engines (default) */
  uint32_t flush_max_writers;       /* concurrent pwrite jobs (default 3); 0 = no limit beyond flush_threads */
  uint64_t flush_write_piece;       /* max bytes per pwrite job (default 32 MiB) */
} lzckpt_engine_config;
void lzckpt_engine_config_defaults(lzckpt_engine_config* c);

typedef struct lzckpt_engine lzckpt_engine;
typedef struct lzckpt_ticket lzckpt_ticket;
int lzckpt_engine_create(const lzckpt_engine_config* c, const lzckpt_topology* topo, uint32_t rank_dp,
                         uint32_t rank_pp, uint32_t rank_tp, lzckpt_engine** out);
void lzckpt_engine_destroy(lzckpt_engine* e);
/* plan = plan_checkpoint(engine topology, *model, step) */
int lzckpt_engine_capture(lzckpt_engine* e, const lzckpt_model_spec* model, const lzckpt_tree* t,
                          uint64_t step, lzckpt_ticket** out);
/* Engine::capture(plan, tree, step, producer_stream): the same capture,
 * ordered on the device after the work already queued on the trainer's
 * `cuda_stream` (a cudaStream_t; NULL = the legacy default stream), so the
 * snapshot never reads a tensor the trainer is still writing. The host does
 * not wait; inline leaves are read behind the producer too. The reference
 * orders reads after writes with its region mutex (transfer_engine.cpp:10-36). */
int lzckpt_engine_capture_on_stream(lzckpt_engine* e, const lzckpt_model_spec* model, const lzckpt_tree* t,
                                    uint64_t step, void* cuda_stream, lzckpt_ticket** out);
int lzckpt_engine_update_barrier(lzckpt_engine* e, lzckpt_ticket* k);
int lzckpt_engine_update_barrier_on_stream(lzckpt_engine* e, lzckpt_ticket* k, void* cuda_stream);
int lzckpt_engine_wait_persisted(lzckpt_engine* e, lzckpt_ticket* k);
int lzckpt_engine_drain(lzckpt_engine* e);
int lzckpt_engine_restore(lzckpt_engine* e, const lzckpt_manifest* m, uint64_t step, lzckpt_tree** out);
int lzckpt_engine_restore_into(lzckpt_engine* e, const lzckpt_manifest* m, uint64_t step, lzckpt_tree* t);
/* Two-phase commit of a persisted capture (CommitCoordinator::run_step with
 * this engine as the participant; reference consolidation.cpp:160-284): the
 * files are validated (header, extent, entry checksums) and their whole-file
 * digests recorded in the manifest, each file read once and hashed on the
 * GPU. Single-rank topologies. *committed = 1 when the step committed, else
 * `reason` says why. */
int lzckpt_engine_commit(lzckpt_engine* e, const lzckpt_model_spec* model, lzckpt_ticket* t, lzckpt_manifest* m,
                         int* committed, char* reason, uint64_t reason_cap);
/* Restore/commit keep their pinned + device stream windows (3 x 512 MiB each)
 * pooled for the next call; this frees the idle ones. */
void lzckpt_trim_caches(void);
/* NUMA placement. Each engine places its pinned ring on
 * its GPU's NUMA node (MPOL_PREFERRED before first touch, by that node's
 * CPUs) and binds its issuer, completion, flush and streamer threads there;
 * lzckpt_engine_numa_node reports the node (-1 = none: single-node host).
 * The helpers below expose the same policy for tests and tools. */
int lzckpt_numa_node_count(void);
int lzckpt_numa_prefer_range(void* p, uint64_t len, int node);
/* Node of each page at p + k*stride (move_pages query), k < cap; *n = pages. */
int lzckpt_numa_page_nodes(const void* p, uint64_t len, uint64_t stride, int* nodes, uint64_t cap, uint64_t* n);
int lzckpt_engine_numa_node(const lzckpt_engine* e);
/* Uplink relay counters: bytes this engine delegated to its helper (owner),
 * bytes and requests it relayed for owners (helper). */
int lzckpt_engine_relay_stats(const lzckpt_engine* e, uint64_t* delegated_bytes, uint64_t* served_bytes,
                              uint64_t* served_requests);
/* Engine::set_relay: delegate `share` of each shard file's payload to the
 * helper serving `peer_socket` (share 0: off); call between captures. */
int lzckpt_engine_set_relay(lzckpt_engine* e, const char* peer_socket, double share);
/* Phase one of the 2PC for THIS rank only (EngineCommitParticipant::prepare,
 * reference consolidation.cpp:142-152): waits until the capture is persisted,
 * then validates the rank's files on the GPU. Writes a JSON vote
 * {"rank","step","vote":"prepared"|"failed","detail","files":[[path,length,digest]]}
 * into `json` when `cap` >= *needed (always set). Multi-process jobs gather
 * these votes over their own transport (paper_2406_10707_b200/commit.py). */
int lzckpt_engine_prepare(lzckpt_engine* e, const lzckpt_model_spec* model, lzckpt_ticket* t, char* json,
                          uint64_t cap, uint64_t* needed);
/* FNV-1a-64 and length of a whole file (the manifest digest), on the GPU. */
int lzckpt_file_digest(const char* path, int device, uint64_t* length, uint64_t* digest);

typedef struct lzckpt_counters {
  uint64_t captures;
  uint64_t bytes_captured;
  double capture_seconds;
  double barrier_seconds;
  double last_capture_seconds;
  double last_barrier_seconds;
} lzckpt_counters;
int lzckpt_engine_counters(const lzckpt_engine* e, lzckpt_counters* out);

typedef struct lzckpt_snapshot_stats {
  uint64_t kernel_launches;
  uint64_t kernel_bytes;
  uint64_t ce_copies;
  uint64_t ce_bytes;
  uint64_t blob_bytes;
  uint64_t groups;
} lzckpt_snapshot_stats;
int lzckpt_engine_snapshot_stats(const lzckpt_engine* e, lzckpt_snapshot_stats* out);
/* bytes the flush pipeline has written, files it persisted */
int lzckpt_engine_flush_stats(const lzckpt_engine* e, uint64_t* bytes_written, uint64_t* files_persisted);
/* Framework glue (DeepSpeed-style checkpoint engine): one LZCKPT01 file for
 * every leaf of the tree, same lazy snapshot path, no plan. */
int lzckpt_engine_capture_file(lzckpt_engine* e, const char* path, const lzckpt_tree* t, uint64_t step,
                               lzckpt_ticket** out);
int lzckpt_engine_capture_file_on_stream(lzckpt_engine* e, const char* path, const lzckpt_tree* t, uint64_t step,
                                         void* cuda_stream, lzckpt_ticket** out);
/* Reads one file back (validated). Region leaves are DMA'd into the
 * same-path, same-size regions of `into` (may be NULL), else fresh regions. */
int lzckpt_engine_restore_file(lzckpt_engine* e, const char* path, const lzckpt_tree* into, lzckpt_tree** out);
/* Finalized header of the ticket's i-th file (checksums as written / hashed). */
int lzckpt_engine_ticket_header(const lzckpt_engine* e, const lzckpt_ticket* k, uint32_t i, lzckpt_header** out);
/* Switches the D2H variant for later captures (B200 tuning knob). */
int lzckpt_engine_set_copy_variant(lzckpt_engine* e, uint64_t ce_threshold, int force_kernel, int force_copy_engine,
                                   uint32_t kernel_ctas, uint64_t group_bytes);
/* the engine's snapshot stream (cudaStream_t) */
void* lzckpt_engine_snapshot_stream(const lzckpt_engine* e);

/* ---- tickets ------------------------------------------------------------------- */
void lzckpt_ticket_release(lzckpt_ticket* k);
uint64_t lzckpt_ticket_id(const lzckpt_ticket* k);
uint64_t lzckpt_ticket_step(const lzckpt_ticket* k);
/* 0 InFlight, 1 HostResident, 2 Persisted, 3 Failed */
int lzckpt_ticket_status(const lzckpt_ticket* k);
int lzckpt_ticket_torn(const lzckpt_ticket* k);
uint64_t lzckpt_ticket_payload_bytes(const lzckpt_ticket* k);
uint32_t lzckpt_ticket_file_count(const lzckpt_ticket* k);
int lzckpt_ticket_file(const lzckpt_ticket* k, uint32_t i, char* path, uint64_t cap);
int lzckpt_ticket_failure_reason(const lzckpt_ticket* k, char* out, uint64_t cap);
/* Device time (ms) of the ticket's D2H snapshot, first device op to last
 * completion on the snapshot stream; < 0 until the copies completed. */
double lzckpt_engine_ticket_device_ms(const lzckpt_engine* e, const lzckpt_ticket* k);

/* ---- synthetic workloads (tests / bench) ------------------------------------- */
/* Materializes the spec written by paper_2406_10707_b200/workloads.py on
 * `device`: *tree gets every leaf, *model / *topo / rank / *step the plan
 * inputs. splitmix64 leaves are generated on the GPU. */
int lzckpt_workload_build(const char* spec_path, int device, lzckpt_tree** tree, lzckpt_model_spec* model,
                          lzckpt_topology* topo, uint32_t rank[3], uint64_t* step, uint64_t* bytes);

#ifdef __cplusplus
}
#endif
#endif /* LZCKPT_C_H_ */
