/*
 * ORACLE — TEST INFRASTRUCTURE ONLY. Never linked into, loaded by, or called
 * from the product (paper_2406_10707_b200/). Only tests/, __graft_entry__.smoke()
 * and bench.py's CPU-baseline leg may use it, and only as the checker.
 *
 * Plain-C restatement of the reference's snapshot-path algorithms, each
 * function citing the reference file:line it follows (paths relative to
 * /root/reference/proj/core). Parity is PINNED: tests/test_oracle.py checks it
 * against the FNV-1a known answers, the reference's golden C1 digests
 * and fixtures produced by running the reference itself
 * (oracle/_ref/ref_snapshot, tests/golden/make_fixtures.py).
 */
#ifndef LZK_ORACLE_H_
#define LZK_ORACLE_H_

#include <stddef.h>
#include <stdint.h>

/* FNV-1a 64 — include/lzckpt/checksum.hpp:17-24 */
uint64_t lzo_fnv1a64(uint64_t state, const uint8_t* p, uint64_t n);

/* Generators (workloads.py) */
void lzo_fill_mt19937_64(uint64_t seed, uint64_t n_leaves, const uint64_t* sizes, uint8_t* const* out);
void lzo_fill_splitmix(uint64_t seed, uint64_t leaf, uint64_t size, uint8_t* out);
/* FNV-1a 64 of the splitmix64 stream of (seed, leaf, size), without storing
 * it (full-size checksum parity of GB-scale shards). */
uint64_t lzo_splitmix_fnv(uint64_t seed, uint64_t leaf, uint64_t size);

/* Ring placement state machine — src/ring_core.cpp:21-139 */
typedef struct lzo_ring lzo_ring;
lzo_ring* lzo_ring_new(uint64_t capacity);
void lzo_ring_free(lzo_ring* r);
/* 1 and (*id,*offset) on success, 0 when nothing fits */
int lzo_ring_try_reserve(lzo_ring* r, uint64_t size, uint64_t* id, uint64_t* offset);
/* 0 ok, -1 illegal transition */
int lzo_ring_mark_filled(lzo_ring* r, uint64_t id);
int lzo_ring_begin_flush(lzo_ring* r, uint64_t id);
int lzo_ring_release(lzo_ring* r, uint64_t id);
uint64_t lzo_ring_live_bytes(const lzo_ring* r);

/* Header size and bytes — src/format.cpp:79-83, :98-115 */
uint64_t lzo_header_size(uint32_t n, const uint32_t* key_lens);
uint64_t lzo_header_serialize(uint32_t n, const char* const* keys, const uint32_t* key_lens,
                              const uint64_t* offsets, const uint64_t* lengths,
                              const uint64_t* checksums, uint8_t* out);

/* Flatten order — src/state_tree.cpp:103-120 (std::map per path component):
 * writes a permutation `order` that sorts the '/'-separated paths. */
void lzo_flatten_order(uint32_t n, const char* const* paths, uint32_t* order);

/* One shard file, byte for byte — src/engine.cpp:96-231 (meta + header
 * layout), src/state_tree.cpp:195-210 (meta codec), src/flush_pipeline.cpp:
 * 194-263 (payload at header_size+offset, per-entry FNV, header last).
 * Leaves must be given in flatten order with their full paths. Returns the
 * file size; writes the file into `out` when non-NULL. */
uint64_t lzo_compose_shard(uint32_t n, const char* const* paths, const uint8_t* is_region,
                           const uint64_t* sizes, const uint8_t* const* data, uint64_t threshold,
                           uint8_t* out);

/* plan_checkpoint for one rank — src/topology.cpp:100-185. Returns the
 * number of shards (0..2); per shard: kind (0 layers, 1 optimizer), size,
 * first layer, layer count, partition. */
int lzo_plan_rank(uint32_t dp, uint32_t pp, uint32_t tp, uint64_t params, uint32_t layers, uint32_t bpp_model,
                  uint32_t bpp_opt, uint32_t flat_rank, uint32_t* kind, uint64_t* size, uint32_t* first_layer,
                  uint32_t* layer_count, uint32_t* partition);

#endif /* LZK_ORACLE_H_ */
