// C ABI over the lzckpt C++ engine; see include/lzckpt_c.h. Every entry point
// catches the C++ exception hierarchy and maps each class to its own code.
#include "lzckpt_c.h"

#include <cstring>
#include <memory>
#include <optional>
#include <string>
#include <vector>

#include "lzckpt/consolidation.hpp"
#include <json.hpp>
#include "lzckpt/engine.hpp"
#include "lzckpt/errors.hpp"
#include "../src/numa.hpp"
#include "lzckpt/format.hpp"
#include "lzckpt/manifest.hpp"
#include "lzckpt/ring_core.hpp"
#include "lzckpt/state_tree.hpp"
#include "lzckpt/topology.hpp"
#include "lzckpt/workload.hpp"
#include "lzk_cuda.h"
#include "../src/file_stream.hpp"

using namespace lzckpt;

struct lzckpt_ring {
  RingCore core;
  explicit lzckpt_ring(uint64_t cap) : core(cap) {}
};
struct lzckpt_header {
  CheckpointFileHeader h;
};
struct lzckpt_region {
  std::shared_ptr<DeviceRegion> r;
};
struct lzckpt_tree {
  StateTree t;
  mutable std::optional<std::vector<StateTree::FlatLeaf>> flat;  // flatten() cache
};
struct lzckpt_manifest {
  std::unique_ptr<ManifestStore> m;
};
struct lzckpt_engine {
  std::unique_ptr<Engine> e;
  ParallelTopology topo;
};
struct lzckpt_ticket {
  std::shared_ptr<CaptureTicket> k;
};

namespace {

thread_local std::string g_err;

template <class Fn>
int guard(Fn&& fn) {
  try {
    fn();
    return LZCKPT_OK;
  } catch (const TornSnapshot& e) {
    g_err = e.what();
    return LZCKPT_E_TORN;
  } catch (const SizeExceedsCapacity& e) {
    g_err = e.what();
    return LZCKPT_E_SIZE_EXCEEDS;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return LZCKPT_E_CONFIG;
  } catch (const WaitTimeout& e) {
    g_err = e.what();
    return LZCKPT_E_WAIT_TIMEOUT;
  } catch (const IllegalTransition& e) {
    g_err = e.what();
    return LZCKPT_E_ILLEGAL_TRANSITION;
  } catch (const DuplicatePath& e) {
    g_err = e.what();
    return LZCKPT_E_DUPLICATE_PATH;
  } catch (const BadMagic& e) {
    g_err = e.what();
    return LZCKPT_E_BAD_MAGIC;
  } catch (const TruncatedFile& e) {
    g_err = e.what();
    return LZCKPT_E_TRUNCATED;
  } catch (const ChecksumMismatch& e) {
    g_err = e.what();
    return LZCKPT_E_CHECKSUM;
  } catch (const FormatError& e) {
    g_err = e.what();
    return LZCKPT_E_FORMAT;
  } catch (const NotCommitted& e) {
    g_err = e.what();
    return LZCKPT_E_NOT_COMMITTED;
  } catch (const CorruptManifest& e) {
    g_err = e.what();
    return LZCKPT_E_CORRUPT_MANIFEST;
  } catch (const IoError& e) {
    g_err = e.what();
    return LZCKPT_E_IO;
  } catch (const DeviceError& e) {
    g_err = e.what();
    return LZCKPT_E_DEVICE;
  } catch (const Error& e) {
    g_err = e.what();
    return LZCKPT_E_ERROR;
  } catch (const std::exception& e) {
    g_err = e.what();
    return LZCKPT_E_INVALID;
  } catch (...) {
    g_err = "unknown exception";
    return LZCKPT_E_INVALID;
  }
}

void need(const void* p, const char* what) {
  if (!p) throw std::invalid_argument(std::string("null ") + what);
}

void copy_str(const std::string& s, char* out, uint64_t cap) {
  if (!out || cap == 0) return;
  const size_t n = std::min<uint64_t>(s.size(), cap - 1);
  std::memcpy(out, s.data(), n);
  out[n] = '\0';
}

ModelSpec to_model(const lzckpt_model_spec* m) {
  ModelSpec s;
  s.param_count = m->param_count;
  s.layer_count = m->layer_count;
  s.hidden_dim = m->hidden_dim;
  s.bytes_per_param_model = m->bytes_per_param_model;
  s.bytes_per_param_optimizer = m->bytes_per_param_optimizer;
  return s;
}

ParallelTopology to_topo(const lzckpt_topology* t) {
  return ParallelTopology{t->dp, t->pp, t->tp, t->gpus_per_node, t->node_count};
}

std::span<const std::byte> bytes_of(const void* p, uint64_t n) {
  return {static_cast<const std::byte*>(p), size_t(n)};
}

}  // namespace

extern "C" {

const char* lzckpt_last_error(void) { return g_err.c_str(); }

const char* lzckpt_build_info(void) {
  return "lzckpt-b200: sm_100a gather kernel + copy-engine D2H, pinned mapped ring, parallel flush";
}

uint64_t lzckpt_fnv1a64(const void* data, uint64_t len) { return fnv64(data, len); }
uint64_t lzckpt_fnv1a64_update(uint64_t state, const void* data, uint64_t len) {
  return Fnv64::fold(state, data, len);
}

// ---- ring -------------------------------------------------------------------

int lzckpt_ring_create(uint64_t capacity, lzckpt_ring** out) {
  return guard([&] {
    need(out, "out");
    *out = new lzckpt_ring(capacity);
  });
}
void lzckpt_ring_destroy(lzckpt_ring* r) { delete r; }
int lzckpt_ring_try_reserve(lzckpt_ring* r, uint64_t size, uint64_t ticket, uint64_t* id, uint64_t* offset) {
  return guard([&] {
    need(r, "ring");
    auto s = r->core.try_reserve(size, ticket);
    if (id) *id = s ? s->id : 0;
    if (offset) *offset = s ? s->offset : 0;
  });
}
int lzckpt_ring_mark_filled(lzckpt_ring* r, uint64_t id) {
  return guard([&] { need(r, "ring"), r->core.mark_filled(id); });
}
int lzckpt_ring_begin_flush(lzckpt_ring* r, uint64_t id) {
  return guard([&] { need(r, "ring"), r->core.begin_flush(id); });
}
int lzckpt_ring_release(lzckpt_ring* r, uint64_t id) {
  return guard([&] { need(r, "ring"), r->core.release(id); });
}
uint64_t lzckpt_ring_live_bytes(const lzckpt_ring* r) { return r ? r->core.live_bytes() : 0; }
uint64_t lzckpt_ring_live_segments(const lzckpt_ring* r) { return r ? r->core.live_segments() : 0; }
uint64_t lzckpt_ring_released_bytes(const lzckpt_ring* r) { return r ? r->core.released_bytes() : 0; }
int lzckpt_ring_segment(const lzckpt_ring* r, uint64_t id, uint64_t* offset, uint64_t* length, int* state) {
  return guard([&] {
    need(r, "ring");
    const Segment* s = r->core.find(id);
    if (!s) throw IllegalTransition("unknown segment " + std::to_string(id));
    if (offset) *offset = s->offset;
    if (length) *length = s->length;
    if (state) *state = int(s->state);
  });
}

// ---- header -------------------------------------------------------------------

static CheckpointFileHeader to_header(const lzckpt_header_entry* e, uint32_t n, uint32_t version) {
  CheckpointFileHeader h;
  h.format_version = version;
  for (uint32_t i = 0; i < n; ++i) {
    h.entries.push_back(HeaderEntry{std::string(e[i].key, e[i].key_len), e[i].offset, e[i].length, e[i].checksum});
  }
  return h;
}

uint64_t lzckpt_header_serialized_size(const lzckpt_header_entry* e, uint32_t n) {
  uint64_t s = 24;
  for (uint32_t i = 0; i < n; ++i) s += 28 + e[i].key_len;
  return s;
}

int lzckpt_header_serialize(const lzckpt_header_entry* e, uint32_t n, uint32_t version, void* out,
                            uint64_t cap, uint64_t* size) {
  return guard([&] {
    if (n) need(e, "entries");
    auto bytes = serialize_header(to_header(e, n, version));
    if (size) *size = bytes.size();
    if (out && cap >= bytes.size()) std::memcpy(out, bytes.data(), bytes.size());
  });
}

int lzckpt_header_parse(const void* bytes, uint64_t n, lzckpt_header** out) {
  return guard([&] {
    need(out, "out");
    if (n) need(bytes, "bytes");
    *out = new lzckpt_header{parse_header(bytes_of(bytes, n))};
  });
}

int lzckpt_file_read_header(const char* path, lzckpt_header** out) {
  return guard([&] {
    need(path, "path");
    need(out, "out");
    *out = new lzckpt_header{read_header(path)};
  });
}

void lzckpt_header_destroy(lzckpt_header* h) { delete h; }
uint32_t lzckpt_header_count(const lzckpt_header* h) { return h ? uint32_t(h->h.entries.size()) : 0; }
uint32_t lzckpt_header_version(const lzckpt_header* h) { return h ? h->h.format_version : 0; }
uint64_t lzckpt_header_size(const lzckpt_header* h) { return h ? h->h.serialized_size() : 0; }
uint64_t lzckpt_header_payload_end(const lzckpt_header* h) { return h ? h->h.payload_end() : 0; }

int lzckpt_header_entry_at(const lzckpt_header* h, uint32_t i, lzckpt_header_entry* out) {
  return guard([&] {
    need(h, "header");
    need(out, "out");
    const HeaderEntry& e = h->h.entries.at(i);
    *out = lzckpt_header_entry{e.key.data(), uint32_t(e.key.size()), e.offset, e.length, e.checksum};
  });
}

int lzckpt_file_validate(const char* path, const lzckpt_header* h, char* bad_keys, uint64_t cap, uint32_t* n_bad) {
  return guard([&] {
    need(path, "path");
    need(h, "header");
    auto bad = validate_entries(path, h->h);
    std::string joined;
    for (const auto& k : bad) joined += (joined.empty() ? "" : "\n") + k;
    copy_str(joined, bad_keys, cap);
    if (n_bad) *n_bad = uint32_t(bad.size());
  });
}

// ---- plan ---------------------------------------------------------------------

int lzckpt_plan_shards(const lzckpt_topology* topo, const lzckpt_model_spec* model, uint32_t flat_rank,
                       lzckpt_shard* out, uint32_t cap, uint32_t* n) {
  return guard([&] {
    need(topo, "topology");
    need(model, "model");
    CheckpointPlan plan = plan_checkpoint(to_topo(topo), to_model(model), 0);
    const auto& shards = plan.shards(flat_rank);
    if (n) *n = uint32_t(shards.size());
    for (uint32_t i = 0; i < shards.size() && i < cap && out; ++i) {
      const auto& s = shards[i];
      lzckpt_shard& o = out[i];
      o.shard_id = s.shard_id;
      o.kind = s.kind == ShardKind::LayerShard ? 0 : 1;
      o.first_layer = s.first_layer;
      o.layer_count = s.layer_count;
      o.partition = s.partition;
      o.size_bytes = s.size_bytes;
      o.owner_dp = s.owner.dp;
      o.owner_pp = s.owner.pp;
      o.owner_tp = s.owner.tp;
      copy_str(s.filename(), o.filename, sizeof o.filename);
    }
  });
}

// ---- regions --------------------------------------------------------------------

int lzckpt_region_create(int device, uint64_t size, lzckpt_region** out) {
  return guard([&] {
    need(out, "out");
    *out = new lzckpt_region{std::make_shared<DeviceRegion>(size, device)};
  });
}

int lzckpt_region_from_host(int device, const void* bytes, uint64_t size, lzckpt_region** out) {
  return guard([&] {
    need(out, "out");
    if (size) need(bytes, "bytes");
    std::vector<std::byte> v(size);
    if (size) std::memcpy(v.data(), bytes, size);
    *out = new lzckpt_region{std::make_shared<DeviceRegion>(std::move(v), device)};
  });
}

int lzckpt_region_wrap(int device, void* device_ptr, uint64_t size, lzckpt_region** out) {
  return guard([&] {
    need(out, "out");
    *out = new lzckpt_region{DeviceRegion::wrap(device_ptr, size, device)};
  });
}

void lzckpt_region_release(lzckpt_region* r) { delete r; }
uint64_t lzckpt_region_size(const lzckpt_region* r) { return r ? r->r->size() : 0; }
uint64_t lzckpt_region_version(const lzckpt_region* r) { return r ? r->r->version() : 0; }
void* lzckpt_region_device_ptr(const lzckpt_region* r) { return r ? r->r->device_ptr() : nullptr; }
int lzckpt_region_device(const lzckpt_region* r) { return r ? r->r->device() : -1; }

int lzckpt_region_read(const lzckpt_region* r, uint64_t offset, void* out, uint64_t n) {
  return guard([&] {
    need(r, "region");
    if (n) need(out, "out");
    r->r->read_chunk(offset, std::span<std::byte>(static_cast<std::byte*>(out), size_t(n)));
  });
}

int lzckpt_region_write(lzckpt_region* r, uint64_t offset, const void* data, uint64_t n) {
  return guard([&] {
    need(r, "region");
    if (n) need(data, "data");
    r->r->write(offset, bytes_of(data, n));
  });
}

int lzckpt_region_mutate(lzckpt_region* r, const void* data, uint64_t n) {
  return guard([&] {
    need(r, "region");
    if (n != r->r->size()) throw std::invalid_argument("mutate: data size must equal region size");
    r->r->mutate([&](std::span<std::byte> b) {
      if (n) std::memcpy(b.data(), data, n);
    });
  });
}

int lzckpt_region_bump_version(lzckpt_region* r) {
  return guard([&] { need(r, "region"), r->r->bump_version(); });
}

// ---- tree -------------------------------------------------------------------------

int lzckpt_tree_create(lzckpt_tree** out) {
  return guard([&] {
    need(out, "out");
    *out = new lzckpt_tree();
  });
}
void lzckpt_tree_destroy(lzckpt_tree* t) { delete t; }

int lzckpt_tree_set_region(lzckpt_tree* t, const char* path, const lzckpt_region* r) {
  return guard([&] {
    need(t, "tree");
    need(path, "path");
    need(r, "region");
    t->t.set_region(path, r->r);
    t->flat.reset();
  });
}

int lzckpt_tree_set_blob(lzckpt_tree* t, const char* path, const void* bytes, uint64_t n) {
  return guard([&] {
    need(t, "tree");
    need(path, "path");
    if (n) need(bytes, "bytes");
    std::vector<std::byte> v(n);
    if (n) std::memcpy(v.data(), bytes, n);
    t->t.set_blob(path, std::move(v));
    t->flat.reset();
  });
}

uint64_t lzckpt_tree_leaf_count(const lzckpt_tree* t) { return t ? t->t.leaf_count() : 0; }
uint64_t lzckpt_tree_total_bytes(const lzckpt_tree* t) { return t ? t->t.total_leaf_bytes() : 0; }

int lzckpt_tree_leaf(const lzckpt_tree* t, uint64_t i, char* path, uint64_t cap, int* is_region, uint64_t* size) {
  return guard([&] {
    need(t, "tree");
    if (!t->flat) t->flat = t->t.flatten();
    const auto& l = t->flat->at(i);
    copy_str(l.path, path, cap);
    if (is_region) *is_region = l.region != nullptr;
    if (size) *size = l.size;
  });
}

int lzckpt_tree_region_at(const lzckpt_tree* t, const char* path, lzckpt_region** out) {
  return guard([&] {
    need(t, "tree");
    need(path, "path");
    need(out, "out");
    *out = new lzckpt_region{t->t.region_at(path)};
  });
}

int lzckpt_tree_blob_at(const lzckpt_tree* t, const char* path, void* out, uint64_t cap, uint64_t* size) {
  return guard([&] {
    need(t, "tree");
    need(path, "path");
    const auto& b = t->t.blob_at(path);
    if (size) *size = b.size();
    if (out && cap >= b.size() && !b.empty()) std::memcpy(out, b.data(), b.size());
  });
}

// ---- manifest ------------------------------------------------------------------------

int lzckpt_manifest_open(const char* path, lzckpt_manifest** out) {
  return guard([&] {
    need(path, "path");
    need(out, "out");
    *out = new lzckpt_manifest{std::make_unique<ManifestStore>(path)};
  });
}
void lzckpt_manifest_destroy(lzckpt_manifest* m) { delete m; }

int lzckpt_manifest_commit_step(lzckpt_manifest* m, uint64_t step, const char* const* paths,
                                const uint64_t* lengths, const uint64_t* digests, uint32_t n) {
  return guard([&] {
    need(m, "manifest");
    CommittedStep s;
    s.step = step;
    for (uint32_t i = 0; i < n; ++i) {
      s.files.push_back(ManifestFileRecord{paths[i], lengths ? lengths[i] : 0, digests ? digests[i] : 0});
    }
    m->m->commit_step(std::move(s));
  });
}

int lzckpt_manifest_is_committed(const lzckpt_manifest* m, uint64_t step) {
  return m && m->m->is_committed(step) ? 1 : 0;
}

int lzckpt_manifest_latest(const lzckpt_manifest* m, int* has, uint64_t* step) {
  return guard([&] {
    need(m, "manifest");
    auto v = m->m->latest_committed();
    if (has) *has = v.has_value();
    if (step) *step = v.value_or(0);
  });
}

// ---- engine ----------------------------------------------------------------------------

void lzckpt_engine_config_defaults(lzckpt_engine_config* c) {
  if (!c) return;
  const EngineConfig d;
  const SnapshotOptions so;
  *c = lzckpt_engine_config{};
  c->checkpoint_root = nullptr;
  c->host_buffer_bytes = d.host_buffer_bytes;
  c->copy_bandwidth_Bps = 0;  // unpaced: the measured device path
  c->chunk_quantum = d.copy_channel.chunk_quantum;
  c->storage_bandwidth_Bps = d.flush.storage_bandwidth_Bps;
  c->fsync_on_finalize = d.flush.fsync_on_finalize;
  c->flush_threads = 0;
  c->large_leaf_threshold = d.large_leaf_threshold;
  c->reserve_timeout_ms = d.reserve_timeout.count();
  c->device = -1;
  c->ce_threshold = so.ce_threshold;
  c->kernel_ctas = so.kernel_ctas;
  c->group_bytes = so.group_bytes;
  c->force_kernel = 0;
  c->force_copy_engine = 0;
  c->hugepages = 1;
  c->flush_discard = 0;
  c->stream_segment_bytes = 0;
  c->flush_hash_only = 0;
  c->relay_serve_socket = nullptr;
  c->relay_staging_bytes = d.relay.staging_bytes;
  c->relay_ctas = d.relay.ctas;
  c->relay_peer_socket = nullptr;
  c->relay_share = 0;
  c->relay_min_entry = d.relay.min_entry;
  c->relay_kernel_route = d.relay.copy_engines ? 0 : 1;
  c->flush_max_writers = d.flush.max_writers;
  c->flush_write_piece = d.flush.write_piece;
}

int lzckpt_engine_create(const lzckpt_engine_config* c, const lzckpt_topology* topo, uint32_t rank_dp,
                         uint32_t rank_pp, uint32_t rank_tp, lzckpt_engine** out) {
  return guard([&] {
    need(c, "config");
    need(topo, "topology");
    need(out, "out");
    EngineConfig cfg;
    cfg.checkpoint_root = c->checkpoint_root ? c->checkpoint_root : "";
    cfg.host_buffer_bytes = c->host_buffer_bytes;
    cfg.copy_channel = ThrottledChannel{c->copy_bandwidth_Bps, c->chunk_quantum};
    cfg.flush.storage_bandwidth_Bps = c->storage_bandwidth_Bps;
    cfg.flush.fsync_on_finalize = c->fsync_on_finalize != 0;
    cfg.flush.threads = c->flush_threads;
    cfg.large_leaf_threshold = c->large_leaf_threshold;
    cfg.reserve_timeout = std::chrono::milliseconds(c->reserve_timeout_ms);
    cfg.snapshot.device = c->device;
    cfg.snapshot.ce_threshold = c->ce_threshold;
    cfg.snapshot.kernel_ctas = c->kernel_ctas;
    cfg.snapshot.group_bytes = c->group_bytes;
    cfg.snapshot.force_kernel = c->force_kernel != 0;
    cfg.snapshot.force_copy_engine = c->force_copy_engine != 0;
    cfg.pool.hugepages = c->hugepages != 0;
    cfg.flush.discard = c->flush_discard != 0;
    cfg.stream_segment_bytes = c->stream_segment_bytes;
    cfg.flush.hash_only = c->flush_hash_only != 0;
    cfg.relay.serve_socket = c->relay_serve_socket ? c->relay_serve_socket : "";
    cfg.relay.staging_bytes = c->relay_staging_bytes;
    cfg.relay.ctas = c->relay_ctas;
    cfg.relay.peer_socket = c->relay_peer_socket ? c->relay_peer_socket : "";
    cfg.relay.share = c->relay_share;
    cfg.relay.min_entry = c->relay_min_entry;
    cfg.relay.copy_engines = c->relay_kernel_route == 0;
    cfg.flush.max_writers = c->flush_max_writers;
    if (c->flush_write_piece) cfg.flush.write_piece = c->flush_write_piece;
    auto h = std::make_unique<lzckpt_engine>();
    h->topo = to_topo(topo);
    h->e = std::make_unique<Engine>(std::move(cfg), h->topo, RankCoord{rank_dp, rank_pp, rank_tp});
    *out = h.release();
  });
}

void lzckpt_engine_destroy(lzckpt_engine* e) { delete e; }

int lzckpt_engine_capture(lzckpt_engine* e, const lzckpt_model_spec* model, const lzckpt_tree* t, uint64_t step,
                          lzckpt_ticket** out) {
  return guard([&] {
    need(e, "engine");
    need(model, "model");
    need(t, "tree");
    need(out, "out");
    CheckpointPlan plan = plan_checkpoint(e->topo, to_model(model), step);
    *out = new lzckpt_ticket{e->e->capture(plan, t->t, step)};
  });
}

int lzckpt_engine_capture_on_stream(lzckpt_engine* e, const lzckpt_model_spec* model, const lzckpt_tree* t,
                                    uint64_t step, void* cuda_stream, lzckpt_ticket** out) {
  return guard([&] {
    need(e, "engine");
    need(model, "model");
    need(t, "tree");
    need(out, "out");
    CheckpointPlan plan = plan_checkpoint(e->topo, to_model(model), step);
    *out = new lzckpt_ticket{e->e->capture(plan, t->t, step, cuda_stream)};
  });
}

int lzckpt_engine_update_barrier(lzckpt_engine* e, lzckpt_ticket* k) {
  return guard([&] {
    need(e, "engine");
    need(k, "ticket");
    e->e->update_barrier(k->k);
  });
}

int lzckpt_engine_update_barrier_on_stream(lzckpt_engine* e, lzckpt_ticket* k, void* cuda_stream) {
  return guard([&] {
    need(e, "engine");
    need(k, "ticket");
    e->e->update_barrier_on_stream(k->k, cuda_stream);
  });
}

int lzckpt_engine_wait_persisted(lzckpt_engine* e, lzckpt_ticket* k) {
  return guard([&] {
    need(e, "engine");
    need(k, "ticket");
    e->e->wait_persisted(k->k);
  });
}

int lzckpt_engine_drain(lzckpt_engine* e) {
  return guard([&] { need(e, "engine"), e->e->drain(); });
}

int lzckpt_engine_restore(lzckpt_engine* e, const lzckpt_manifest* m, uint64_t step, lzckpt_tree** out) {
  return guard([&] {
    need(e, "engine");
    need(m, "manifest");
    need(out, "out");
    auto t = std::make_unique<lzckpt_tree>();
    t->t = e->e->restore(*m->m, step);
    *out = t.release();
  });
}

int lzckpt_engine_restore_into(lzckpt_engine* e, const lzckpt_manifest* m, uint64_t step, lzckpt_tree* t) {
  return guard([&] {
    need(e, "engine");
    need(m, "manifest");
    need(t, "tree");
    e->e->restore_into(*m->m, step, t->t);
  });
}

int lzckpt_file_digest(const char* path, int device, uint64_t* length, uint64_t* digest) {
  return guard([&] {
    need(path, "path");
    need(length, "length");
    need(digest, "digest");
    auto streamer = detail::FileStreamer::acquire(device);
    *digest = streamer->digest(path, length);
  });
}

void lzckpt_trim_caches(void) { detail::FileStreamer::trim(); }

int lzckpt_numa_node_count(void) { return detail::numa_node_count(); }

int lzckpt_numa_prefer_range(void* p, uint64_t len, int node) {
  return guard([&] {
    need(p, "range");
    if (!detail::prefer_node(p, len, node)) throw Error("mbind(MPOL_PREFERRED) failed");
  });
}

int lzckpt_numa_page_nodes(const void* p, uint64_t len, uint64_t stride, int* nodes, uint64_t cap, uint64_t* n) {
  return guard([&] {
    need(p, "range");
    need(nodes, "nodes");
    const int r = detail::page_nodes(p, len, stride, nodes, cap);
    if (r < 0) throw Error("move_pages query failed: errno " + std::to_string(-r));
    if (n) *n = uint64_t(r);
  });
}

int lzckpt_engine_numa_node(const lzckpt_engine* e) { return e ? e->e->pool().numa_node() : -1; }

int lzckpt_engine_set_relay(lzckpt_engine* e, const char* peer_socket, double share) {
  return guard([&] {
    need(e, "engine");
    e->e->set_relay(peer_socket ? peer_socket : "", share);
  });
}

int lzckpt_engine_relay_stats(const lzckpt_engine* e, uint64_t* delegated_bytes, uint64_t* served_bytes,
                              uint64_t* served_requests) {
  return guard([&] {
    need(e, "engine");
    const auto s = e->e->relay_stats();
    if (delegated_bytes) *delegated_bytes = s.delegated_bytes;
    if (served_bytes) *served_bytes = s.served_bytes;
    if (served_requests) *served_requests = s.served_requests;
  });
}

int lzckpt_engine_prepare(lzckpt_engine* e, const lzckpt_model_spec* model, lzckpt_ticket* t, char* json,
                          uint64_t cap, uint64_t* needed) {
  return guard([&] {
    need(e, "engine");
    need(model, "model");
    need(t, "ticket");
    need(needed, "needed");
    const uint64_t step = t->k->step();
    const CheckpointPlan plan = plan_checkpoint(e->topo, to_model(model), step);
    EngineCommitParticipant part(*e->e, plan, t->k);
    const auto rep = part.prepare(step);  // wait_persisted + GPU validation of this rank's files
    nlohmann::json j;
    j["rank"] = part.flat_rank();
    j["step"] = step;
    j["vote"] = rep && rep->vote == Vote::Prepared ? "prepared" : "failed";
    j["detail"] = rep ? rep->detail : "no answer";
    j["files"] = nlohmann::json::array();
    if (rep) {
      for (const auto& f : rep->files) j["files"].push_back({f.relative_path, f.length, f.digest});
    }
    // leaf keys in `detail` are user strings: never throw on invalid UTF-8
    const std::string out = j.dump(-1, ' ', false, nlohmann::json::error_handler_t::replace);
    *needed = out.size() + 1;
    if (json && cap >= out.size() + 1) std::memcpy(json, out.c_str(), out.size() + 1);
  });
}

int lzckpt_engine_commit(lzckpt_engine* e, const lzckpt_model_spec* model, lzckpt_ticket* t, lzckpt_manifest* m,
                         int* committed, char* reason, uint64_t reason_cap) {
  return guard([&] {
    need(e, "engine");
    need(model, "model");
    need(t, "ticket");
    need(m, "manifest");
    need(committed, "committed");
    if (e->topo.ranks() != 1) {
      throw ConfigError("lzckpt_engine_commit: single-rank topologies only (one participant per process)");
    }
    const uint64_t step = t->k->step();
    const CheckpointPlan plan = plan_checkpoint(e->topo, to_model(model), step);
    EngineCommitParticipant part(*e->e, plan, t->k);
    CommitCoordinator coord(*m->m, e->topo);
    const CommitRecord rec = coord.run_step(step, {&part});
    *committed = rec.decision == Decision::Committed ? 1 : 0;
    if (reason && reason_cap) {
      std::strncpy(reason, rec.reason.c_str(), size_t(reason_cap) - 1);
      reason[reason_cap - 1] = '\0';
    }
  });
}

int lzckpt_engine_counters(const lzckpt_engine* e, lzckpt_counters* out) {
  return guard([&] {
    need(e, "engine");
    need(out, "out");
    auto c = e->e->counters();
    *out = lzckpt_counters{c.captures, c.bytes_captured, c.capture_seconds, c.barrier_seconds,
                           c.last_capture_seconds, c.last_barrier_seconds};
  });
}

int lzckpt_engine_snapshot_stats(const lzckpt_engine* e, lzckpt_snapshot_stats* out) {
  return guard([&] {
    need(e, "engine");
    need(out, "out");
    auto s = e->e->transfers().stats();
    *out = lzckpt_snapshot_stats{s.kernel_launches, s.kernel_bytes, s.ce_copies, s.ce_bytes, s.blob_bytes, s.groups};
  });
}

int lzckpt_engine_flush_stats(const lzckpt_engine* e, uint64_t* bytes_written, uint64_t* files_persisted) {
  return guard([&] {
    need(e, "engine");
    if (bytes_written) *bytes_written = e->e->flush().bytes_written();
    if (files_persisted) *files_persisted = e->e->flush().files_persisted();
  });
}

int lzckpt_engine_capture_file(lzckpt_engine* e, const char* path, const lzckpt_tree* t, uint64_t step,
                               lzckpt_ticket** out) {
  return guard([&] {
    need(e, "engine");
    need(path, "path");
    need(t, "tree");
    need(out, "out");
    *out = new lzckpt_ticket{e->e->capture_file(path, t->t, step)};
  });
}

int lzckpt_engine_capture_file_on_stream(lzckpt_engine* e, const char* path, const lzckpt_tree* t, uint64_t step,
                                         void* cuda_stream, lzckpt_ticket** out) {
  return guard([&] {
    need(e, "engine");
    need(path, "path");
    need(t, "tree");
    need(out, "out");
    *out = new lzckpt_ticket{e->e->capture_file(path, t->t, step, cuda_stream)};
  });
}

int lzckpt_engine_restore_file(lzckpt_engine* e, const char* path, const lzckpt_tree* into, lzckpt_tree** out) {
  return guard([&] {
    need(e, "engine");
    need(path, "path");
    need(out, "out");
    auto t = std::make_unique<lzckpt_tree>();
    t->t = e->e->restore_file(path, into ? &into->t : nullptr);
    *out = t.release();
  });
}

int lzckpt_engine_ticket_header(const lzckpt_engine* e, const lzckpt_ticket* k, uint32_t i, lzckpt_header** out) {
  return guard([&] {
    need(e, "engine");
    need(k, "ticket");
    need(out, "out");
    auto hs = e->e->ticket_headers(k->k);
    *out = new lzckpt_header{hs.at(i)};
  });
}

int lzckpt_engine_set_copy_variant(lzckpt_engine* e, uint64_t ce_threshold, int force_kernel, int force_copy_engine,
                                   uint32_t kernel_ctas, uint64_t group_bytes) {
  return guard([&] {
    need(e, "engine");
    SnapshotOptions o = e->e->transfers().options();
    o.ce_threshold = ce_threshold;
    o.force_kernel = force_kernel != 0;
    o.force_copy_engine = force_copy_engine != 0;
    if (kernel_ctas) o.kernel_ctas = kernel_ctas;
    if (group_bytes) o.group_bytes = group_bytes;
    e->e->transfers().set_options(o);
  });
}

void* lzckpt_engine_snapshot_stream(const lzckpt_engine* e) {
  return e ? lzk_stream_handle(e->e->transfers().stream()) : nullptr;
}

// ---- tickets -----------------------------------------------------------------------------

void lzckpt_ticket_release(lzckpt_ticket* k) { delete k; }
uint64_t lzckpt_ticket_id(const lzckpt_ticket* k) { return k ? k->k->id() : 0; }
uint64_t lzckpt_ticket_step(const lzckpt_ticket* k) { return k ? k->k->step() : 0; }
int lzckpt_ticket_status(const lzckpt_ticket* k) { return k ? int(k->k->status()) : -1; }
int lzckpt_ticket_torn(const lzckpt_ticket* k) { return k && k->k->torn() ? 1 : 0; }
uint64_t lzckpt_ticket_payload_bytes(const lzckpt_ticket* k) { return k ? k->k->payload_bytes() : 0; }
uint32_t lzckpt_ticket_file_count(const lzckpt_ticket* k) { return k ? uint32_t(k->k->shard_files().size()) : 0; }

int lzckpt_ticket_file(const lzckpt_ticket* k, uint32_t i, char* path, uint64_t cap) {
  return guard([&] {
    need(k, "ticket");
    copy_str(k->k->shard_files().at(i).string(), path, cap);
  });
}

double lzckpt_engine_ticket_device_ms(const lzckpt_engine* e, const lzckpt_ticket* k) {
  return e && k ? e->e->transfers().ticket_device_ms(k->k->id()) : -1.0;
}

int lzckpt_ticket_failure_reason(const lzckpt_ticket* k, char* out, uint64_t cap) {
  return guard([&] {
    need(k, "ticket");
    copy_str(k->k->failure_reason(), out, cap);
  });
}

// ---- workloads ------------------------------------------------------------------------------

int lzckpt_workload_build(const char* spec_path, int device, lzckpt_tree** tree, lzckpt_model_spec* model,
                          lzckpt_topology* topo, uint32_t rank[3], uint64_t* step, uint64_t* bytes) {
  return guard([&] {
    need(spec_path, "spec");
    need(tree, "tree");
    Workload w = build_workload(spec_path, device);
    auto t = std::make_unique<lzckpt_tree>();
    t->t = std::move(w.tree);
    if (model) {
      *model = lzckpt_model_spec{w.model.param_count, w.model.layer_count, w.model.hidden_dim,
                                 w.model.bytes_per_param_model, w.model.bytes_per_param_optimizer};
    }
    if (topo) *topo = lzckpt_topology{w.topo.dp, w.topo.pp, w.topo.tp, w.topo.gpus_per_node, w.topo.node_count};
    if (rank) {
      rank[0] = w.rank.dp;
      rank[1] = w.rank.pp;
      rank[2] = w.rank.tp;
    }
    if (step) *step = w.step;
    if (bytes) *bytes = w.bytes;
    *tree = t.release();
  });
}

}  // extern "C"
