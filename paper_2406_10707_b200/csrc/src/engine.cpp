// Per-rank lazy snapshot engine; see include/lzckpt/engine.hpp.
//
// Reference flow reproduced (proj/core/src/engine.cpp):
//   capture: positional plan/tree match, per-shard flatten + size check,
//   small leaves captured synchronously into __meta__, header offsets dense
//   from serialized_size, one ring segment per shard file, file registered,
//   [meta, large...] copy tasks submitted                       :96-231
//   update_barrier / wait_persisted / drain                     :233-267
//   on_file_done / on_torn / ticket_status / counters           :269-328
//   read_entry / restore                                        :330-379
// B200 changes: all small region leaves of a capture are snapshotted by ONE
// gather launch into pinned staging (the reference pays one locked clone per
// leaf); restore streams each file once through pinned windows (the
// reference reads it three times), hashing entries in parallel and DMAing
// them into fresh HBM regions while the next window is read.
#include "lzckpt/engine.hpp"

#include <fcntl.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cerrno>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <utility>

#include "file_stream.hpp"
#include "lzckpt/errors.hpp"
#include "lzk_cuda.h"
#include "numa.hpp"
#include "relay.hpp"

namespace lzckpt {

using detail::ck;
using detail::EntrySink;
using detail::FileStreamer;
using detail::PhaseTrace;
using detail::since;

namespace {

// Large leaves are placed 4 KiB-aligned in the pinned ring when the capture
// is big enough to matter: the payload starts `pad` bytes into a segment
// reserved with 4 KiB of slack, so that ring address + __meta__ size is
// aligned (C2 tensors are 4 KiB multiples, so every one of them lands
// aligned). Copy engines on some B200 hosts lose 7-8 % on misaligned
// destinations (tools/dma_gap.py); file offsets are unchanged.
constexpr uint64_t kRingAlign = 4096;
constexpr uint64_t kAlignMin = 16ull << 20;

uint64_t aligned_pad(const std::byte* seg_base, uint64_t meta_size, uint64_t payload_offset) {
  const uint64_t a = reinterpret_cast<uint64_t>(seg_base) + meta_size - payload_offset;  // mod 2^64
  return (kRingAlign - a % kRingAlign) % kRingAlign;
}

struct ShardBuild {
  uint64_t shard_id = 0;
  std::filesystem::path path;
  CheckpointFileHeader header;
  std::shared_ptr<const std::byte> meta;  // pinned, mapped (MetaPool)
  uint64_t meta_size = 0;
  struct Large {
    StateTree::RegionPtr region;
    StateTree::BlobPtr blob;
    uint64_t size = 0;
  };
  std::vector<Large> larges;
  uint64_t payload = 0;
};

// Pinned staging buffer that grows on demand.
struct Pinned {
  std::byte* p = nullptr;
  uint64_t cap = 0;
  ~Pinned() { lzk_host_free(p); }
  void ensure(uint64_t n) {
    if (n <= cap) return;
    lzk_host_free(p);
    p = nullptr;
    cap = 0;
    void* q = nullptr;
    ck(lzk_host_alloc(std::max<uint64_t>(n, 1), LZK_HOST_MAPPED | LZK_HOST_HUGEPAGE, &q), "pinned staging");
    p = static_cast<std::byte*>(q);
    cap = n;
  }
};

}  // namespace


const char* to_string(TicketStatus s) {
  switch (s) {
    case TicketStatus::InFlight: return "in-flight";
    case TicketStatus::HostResident: return "host-resident";
    case TicketStatus::Persisted: return "persisted";
    case TicketStatus::Failed: return "failed";
  }
  return "?";
}

TicketStatus CaptureTicket::status() const {
  std::lock_guard lk(mu_);
  if (engine_) return engine_->ticket_status(*this);
  if (failed_) return TicketStatus::Failed;
  if (files_done_ == files_.size()) return TicketStatus::Persisted;
  return barrier_passed_ ? TicketStatus::HostResident : TicketStatus::InFlight;
}

bool CaptureTicket::torn() const {
  std::lock_guard lk(mu_);
  return torn_;
}

std::string CaptureTicket::failure_reason() const {
  std::lock_guard lk(mu_);
  return failure_reason_;
}

std::vector<std::filesystem::path> CaptureTicket::shard_files() const {
  std::lock_guard lk(mu_);
  std::vector<std::filesystem::path> out;
  for (const auto& f : files_) out.push_back(f.path);
  return out;
}

Engine::Engine(EngineConfig config, ParallelTopology topo, RankCoord rank)
    : config_(std::move(config)),
      topo_(topo),
      rank_(rank),
      pool_(config_.host_buffer_bytes, config_.reserve_timeout,
            [this] {
              PoolOptions o = config_.pool;
              if (o.device < 0) o.device = config_.snapshot.device;
              return o;
            }()),
      transfers_(pool_, config_.copy_channel, config_.snapshot),
      flush_(pool_, config_.flush) {
  topo_.validate();
  if (config_.checkpoint_root.empty()) throw ConfigError("checkpoint root not set");
  if (config_.large_leaf_threshold == 0) throw ConfigError("large-leaf threshold must be > 0");
  ck(lzk_stream_create(transfers_.device(), 0, &inline_stream_), "inline snapshot stream");
  transfers_.set_chunk_callback([this](uint64_t seg, uint64_t off, uint64_t len) {
    flush_.enqueue_flush(seg, off, len);  // paced path
  });
  transfers_.set_span_callback([this](const std::vector<ChunkSpan>& spans) { flush_.enqueue_flush_spans(spans); });
  transfers_.set_torn_callback([this](const CopyTask& t) { on_torn(t.ticket); });
  if (config_.stream_segment_bytes > 0) {
    if (config_.stream_segment_bytes > config_.host_buffer_bytes) {
      throw ConfigError("stream_segment_bytes exceeds the host buffer pool");
    }
    streamer_ = std::thread([this] { streamer_loop(); });
  }
  if (!config_.relay.serve_socket.empty()) {
    relay_server_ = std::make_unique<detail::RelayServer>(transfers_.device(), config_.relay.serve_socket,
                                                          config_.relay.staging_bytes, config_.relay.ctas,
                                                          config_.relay.copy_engines);
  }
  if (!config_.relay.peer_socket.empty() && config_.relay.share > 0) set_relay(config_.relay.peer_socket, config_.relay.share);
}

Engine::~Engine() {
  try {
    drain();
  } catch (...) {
  }
  {
    std::lock_guard lk(stream_mu_);
    stream_stop_ = true;
  }
  stream_cv_.notify_all();
  if (streamer_.joinable()) streamer_.join();
  {
    std::lock_guard lk(mu_);
    for (auto& [id, weak] : tickets_) {
      if (auto t = weak.lock()) {
        std::lock_guard tl(t->mu_);
        t->engine_ = nullptr;
      }
    }
  }
  relay_client_.reset();  // after drain(): every delegated file has completed
  relay_server_.reset();
  for (auto& [e, h] : relay_events_) lzk_event_destroy(e);
  lzk_stream_destroy(inline_stream_);
}

struct Engine::MetaPool {
  std::mutex mu;
  std::vector<std::pair<std::byte*, uint64_t>> free;  // pinned blocks, capacity
  ~MetaPool() {
    for (auto& [p, n] : free) lzk_host_free(p);
  }
};

std::shared_ptr<const std::byte> Engine::meta_buffer(uint64_t bytes) {
  if (!meta_pool_) meta_pool_ = std::make_shared<MetaPool>();
  std::byte* p = nullptr;
  uint64_t cap = 0;
  {
    std::lock_guard lk(meta_pool_->mu);
    auto& fl = meta_pool_->free;  // best fit
    size_t best = fl.size();
    for (size_t i = 0; i < fl.size(); ++i) {
      if (fl[i].second >= bytes && (best == fl.size() || fl[i].second < fl[best].second)) best = i;
    }
    if (best < fl.size()) {
      std::tie(p, cap) = fl[best];
      fl.erase(fl.begin() + long(best));
    }
  }
  if (!p) {
    cap = std::max<uint64_t>(bytes, 1);
    void* q = nullptr;
    ck(lzk_host_alloc(cap, LZK_HOST_MAPPED, &q), "meta buffer");
    p = static_cast<std::byte*>(q);
  }
  auto pool = meta_pool_;  // the buffer may outlive the engine (tickets detach)
  return std::shared_ptr<const std::byte>(p, [pool, cap](const std::byte* q) {
    std::lock_guard lk(pool->mu);
    if (pool->free.size() < 8) {
      pool->free.emplace_back(const_cast<std::byte*>(q), cap);
    } else {
      lzk_host_free(const_cast<std::byte*>(q));
    }
  });
}

std::vector<Engine::FileSpec> Engine::plan_files(const CheckpointPlan& plan, const StateTree& state,
                                                 uint64_t step) const {
  PhaseTrace ftr("capture-flatten");
  const auto& shards = plan.shards(flat_rank(topo_, rank_));
  const auto names = state.top_level_names();
  if (names.size() != shards.size()) {
    throw ConfigError("state tree has " + std::to_string(names.size()) +
                      " top-level children but the plan assigns " + std::to_string(shards.size()) +
                      " shards to this rank");
  }
  // Validate everything before the first reservation (a rejected capture
  // must not strand a segment).
  std::vector<FileSpec> files(shards.size());
  for (size_t i = 0; i < shards.size(); ++i) {
    files[i].path = shard_path(config_.checkpoint_root, step, shards[i]);
    files[i].shard_id = shards[i].shard_id;
    files[i].leaves = state.flatten_child_shared(names[i]);
    uint64_t sum = 0;
    for (const auto& l : *files[i].leaves) sum += l.size;
    if (sum != shards[i].size_bytes) {
      throw ConfigError("subtree '" + names[i] + "' holds " + std::to_string(sum) + " bytes but shard " +
                        shards[i].filename() + " expects " + std::to_string(shards[i].size_bytes));
    }
  }
  ftr.mark("flatten");
  return files;
}

std::shared_ptr<CaptureTicket> Engine::capture(const CheckpointPlan& plan, const StateTree& state,
                                               uint64_t step) {
  const auto t0 = std::chrono::steady_clock::now();
  auto files = plan_files(plan, state, step);
  return capture_impl(files, step, t0, Producer{});
}

std::shared_ptr<CaptureTicket> Engine::capture(const CheckpointPlan& plan, const StateTree& state,
                                               uint64_t step, void* producer_stream) {
  const auto t0 = std::chrono::steady_clock::now();
  auto files = plan_files(plan, state, step);
  return capture_impl(files, step, t0, Producer{true, producer_stream});
}

namespace {

std::vector<StateTree::FlatLeaf> file_leaves(const StateTree& state) {
  auto leaves = state.flatten();
  if (leaves.empty()) throw ConfigError("capture_file: empty state tree");
  return leaves;
}

}  // namespace

std::shared_ptr<CaptureTicket> Engine::capture_file(const std::filesystem::path& path, const StateTree& state,
                                                    uint64_t step) {
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<FileSpec> files(1);
  files[0].path = path;
  files[0].leaves = std::make_shared<const std::vector<StateTree::FlatLeaf>>(file_leaves(state));
  return capture_impl(files, step, t0, Producer{});
}

std::shared_ptr<CaptureTicket> Engine::capture_file(const std::filesystem::path& path, const StateTree& state,
                                                    uint64_t step, void* producer_stream) {
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<FileSpec> files(1);
  files[0].path = path;
  files[0].leaves = std::make_shared<const std::vector<StateTree::FlatLeaf>>(file_leaves(state));
  return capture_impl(files, step, t0, Producer{true, producer_stream});
}

std::shared_ptr<CaptureTicket> Engine::capture_impl(std::vector<FileSpec>& files, uint64_t step,
                                                    std::chrono::steady_clock::time_point t0, Producer producer) {
  detail::NvtxRange range("lzckpt.capture");
  PhaseTrace tr;
  std::vector<ShardBuild> builds(files.size());
  for (auto& f : files) {
    for (const auto& l : *f.leaves) {
      if (l.path == StateTree::kMetaKey) {
        throw DuplicatePath("top-level leaf name '" + l.path + "' is reserved");
      }
      if (l.region && l.region->device() != transfers_.device()) {
        throw ConfigError("leaf '" + l.path + "' lives on device " + std::to_string(l.region->device()) +
                          ", engine on " + std::to_string(transfers_.device()));
      }
    }
  }
  tr.mark("flatten+validate");

  // Ordered capture on the device path: the inline gather becomes the
  // ticket's first device op (after the producer wait) instead of a
  // synchronous launch here. The paced channel is host-driven, so there the
  // inline gather stays synchronous, behind a device-side producer wait.
  const bool deferred_inline = producer.ordered && config_.copy_channel.bandwidth_Bps <= 0;
  std::vector<lzk_copy_desc> inl;
  std::vector<StateTree::RegionPtr> inl_regions;
  {
    std::lock_guard il(inline_mu_);  // one inline gather at a time (inline_stream_)
    // Small region leaves go straight from HBM into their slots of __meta__
    // (pinned, mapped), by ONE gather launch for the whole capture; the
    // reference clones each under a lock (engine.cpp:138-143).
    for (size_t i = 0; i < files.size(); ++i) {
      ShardBuild& b = builds[i];
      b.shard_id = files[i].shard_id;
      b.path = files[i].path;
      const auto& leaves_i = *files[i].leaves;
      // __meta__ in one pass, serialize_leaf_manifest's layout
      // (state_tree.cpp; reference state_tree.cpp:195-210): u32 n, then per
      // leaf u32 len, path, u8 flags (1 region | 2 inlined), u64 size, and
      // the inline bytes (host blobs copied here, regions by the kernel).
      uint64_t total = 4, nlarge = 0;
      for (const auto& l : leaves_i) {
        const bool inl_leaf = l.size < config_.large_leaf_threshold;
        total += 4 + l.path.size() + 1 + 8 + (inl_leaf ? l.size : 0);
        nlarge += inl_leaf ? 0 : 1;
      }
      b.meta = meta_buffer(total);
      b.meta_size = total;
      std::byte* p = const_cast<std::byte*>(b.meta.get());
      auto le = [&p](uint64_t v, int w) {
        for (int k = 0; k < w; ++k) *p++ = std::byte(v >> (8 * k));
      };
      le(leaves_i.size(), 4);
      b.header.entries.reserve(1 + nlarge);
      b.header.entries.push_back({std::string(StateTree::kMetaKey), 0, total, 0});
      b.larges.reserve(nlarge);
      for (const auto& l : leaves_i) {
        const bool inl_leaf = l.size < config_.large_leaf_threshold;
        le(l.path.size(), 4);
        std::memcpy(p, l.path.data(), l.path.size());
        p += l.path.size();
        *p++ = std::byte((l.region ? 1 : 0) | (inl_leaf ? 2 : 0));
        le(l.size, 8);
        if (inl_leaf) {
          if (l.region) {
            if (l.size) {
              inl.push_back({reinterpret_cast<uint64_t>(l.region->device_ptr()), reinterpret_cast<uint64_t>(p), l.size});
              if (deferred_inline) inl_regions.push_back(l.region);
            }
          } else if (l.size) {
            std::memcpy(p, l.blob->data(), l.size);
          }
          p += l.size;
        } else {
          b.larges.push_back({l.region, l.blob, l.size});
          b.header.entries.push_back({l.path, 0, l.size, 0});
        }
      }
      uint64_t cursor = b.header.serialized_size();
      for (auto& e : b.header.entries) {
        e.offset = cursor;
        cursor += e.length;
      }
      b.payload = cursor - b.header.serialized_size();
    }
    tr.mark("meta+header");
    if (!inl.empty() && !deferred_inline) {
      // synchronous: the bytes are captured before capture() returns
      if (producer.ordered) ck(lzk_stream_wait_raw(inline_stream_, producer.stream), "inline gather: producer wait");
      ck(lzk_gather_d2h(inline_stream_, inl.data(), uint32_t(inl.size()), config_.snapshot.kernel_ctas),
         "inline leaf gather");
      ck(lzk_stream_sync(inline_stream_), "inline leaf gather sync");
    }
    tr.mark("inline_gather");
  }

  auto ticket = std::shared_ptr<CaptureTicket>(new CaptureTicket());
  {
    std::lock_guard lk(mu_);
    ticket->id_ = next_ticket_++;
    ticket->step_ = step;
    ticket->rank_ = rank_;
    ticket->engine_ = this;
    std::erase_if(tickets_, [](const auto& kv) { return kv.second.expired(); });
    tickets_.emplace(ticket->id_, ticket);
  }
  if (deferred_inline) {
    std::vector<std::shared_ptr<const void>> keep;
    for (const auto& b : builds) keep.push_back(b.meta);  // the gather writes into every file's __meta__
    transfers_.set_prologue(ticket->id_, producer.stream, std::move(inl), std::move(inl_regions), std::move(keep));
  } else if (producer.ordered) {
    // paced channel: its host-driven reads are ordered by a host wait here
    ck(lzk_stream_wait_raw(inline_stream_, producer.stream), "capture: producer wait");
    ck(lzk_stream_sync(inline_stream_), "capture: producer wait");
  }

  uint64_t total = 0;
  std::weak_ptr<CaptureTicket> weak = ticket;
  if (config_.stream_segment_bytes > 0) {
    // Streaming: cut each file's payload [meta][large...] into segments of at
    // most S bytes; the streamer reserves them in order (backpressure) and
    // submits their copies. File bytes are identical to the one-segment path.
    const uint64_t S = config_.stream_segment_bytes;
    std::vector<StreamJob> jobs;
    for (auto& b : builds) {
      const uint64_t file_id = flush_.register_streamed_file(b.path, std::move(b.header),
                                                             [this, weak](uint64_t, FlushFileState st) {
                                                               if (auto t = weak.lock()) on_file_done(t, st);
                                                             });
      {
        std::lock_guard tl(ticket->mu_);
        ticket->files_.push_back({b.path, file_id, 0});
        ticket->streamed_ = true;
      }
      struct Src {
        StateTree::RegionPtr region;
        StateTree::BlobPtr blob;
        uint64_t size;
      };
      std::vector<Src> srcs{{nullptr, nullptr, b.meta_size}};  // [0] = __meta__ (pinned)
      for (const auto& l : b.larges) srcs.push_back({l.region, l.blob, l.size});
      size_t si = 0;
      uint64_t soff = 0;
      for (uint64_t seg_off = 0; seg_off < b.payload; seg_off += S) {
        StreamJob j;
        j.ticket = ticket;
        j.file_id = file_id;
        j.meta_size = b.meta_size;
        j.payload_offset = seg_off;
        j.length = std::min(S, b.payload - seg_off);
        for (uint64_t filled = 0; filled < j.length;) {
          const Src& src = srcs[si];
          const uint64_t n = std::min(src.size - soff, j.length - filled);
          if (n) {
            auto t = std::make_shared<CopyTask>();
            t->ticket = ticket->id_;
            t->shard_id = b.shard_id;
            t->source.region = src.region;
            if (si == 0) {
              t->source.host_ptr = b.meta.get();
              t->source.host_size = b.meta_size;
              t->source.host_keep = b.meta;
            } else if (!src.region) {
              t->source.host_blob = src.blob;
            }
            t->src_offset = soff;
            t->length = n;
            t->dst_offset = filled;
            j.tasks.push_back(std::move(t));
          }
          filled += n;
          soff += n;
          if (soff == src.size) {
            ++si;
            soff = 0;
          }
        }
        j.tasks.back()->final_for_segment = true;
        jobs.push_back(std::move(j));
      }
      total += b.payload;
    }
    {
      std::lock_guard tl(ticket->mu_);
      ticket->streams_pending_ += jobs.size();
    }
    {
      std::lock_guard sl(stream_mu_);
      for (auto& j : jobs) stream_queue_.push_back(std::move(j));
    }
    stream_cv_.notify_all();
    ticket->payload_bytes_ = total;
    const double dt = since(t0);
    std::lock_guard lk(mu_);
    ++counters_.captures;
    counters_.bytes_captured += total;
    counters_.capture_seconds += dt;
    counters_.last_capture_seconds = dt;
    return ticket;
  }
  double share = 0;
  {
    std::lock_guard lk(relay_mu_);
    share = relay_client_ ? relay_share_ : 0;
  }
  const bool relay = share > 0 && config_.copy_channel.bandwidth_Bps <= 0;
  // the ticket's device time closes only after its last file is submitted
  transfers_.hold(ticket->id_);
  struct Seal {
    TransferEngine& t;
    uint64_t id;
    ~Seal() { t.seal(id); }
  } seal{transfers_, ticket->id_};
  for (auto& b : builds) {
    // Uplink relay: a suffix of the file's large region leaves, up to `share`
    // of its payload, goes to the helper (its bytes never enter this ring).
    size_t own = b.larges.size();
    if (relay) {
      uint64_t moved = 0;
      const uint64_t budget = uint64_t(share * double(b.payload));
      while (own > 0) {
        const auto& l = b.larges[own - 1];
        if (!l.region || l.size < config_.relay.min_entry || moved + l.size > budget) break;
        moved += l.size;
        --own;
      }
    }
    std::vector<std::shared_ptr<DeviceRegion>> relay_regions;
    std::vector<uint64_t> relay_sizes, relay_offsets;
    for (size_t k = own; k < b.larges.size(); ++k) {
      relay_regions.push_back(b.larges[k].region);
      relay_sizes.push_back(b.larges[k].size);
      relay_offsets.push_back(b.header.entries[1 + k].offset);
    }
    const uint64_t header_size = b.header.serialized_size();
    const uint64_t suffix = own < b.larges.size() ? b.header.entries[1 + own].offset - header_size : 0;
    const bool align = b.payload >= kAlignMin && b.payload + kRingAlign <= pool_.capacity();
    const Segment seg = pool_.reserve(b.payload + (align ? kRingAlign - 1 : 0), ticket->id_);  // backpressure
    const uint64_t pad = align ? aligned_pad(pool_.segment_data(seg), b.meta_size, 0) : 0;
    const uint64_t file_id = flush_.register_file(b.path, std::move(b.header), seg.id,
                                                  [this, weak](uint64_t, FlushFileState st) {
                                                    if (auto t = weak.lock()) on_file_done(t, st);
                                                  },
                                                  pad);
    {
      std::lock_guard tl(ticket->mu_);
      ticket->files_.push_back({b.path, file_id, seg.id});
    }
    if (!relay_regions.empty()) {
      flush_.set_external_suffix(file_id, suffix);
      relay_submit(ticket, b.path, file_id, relay_regions, relay_sizes, relay_offsets, producer.stream,
                   producer.ordered);
      b.larges.resize(own);
    }
    // one allocation for the file's tasks; each task shares the block. Tasks
    // are submitted in chunks as they are built, so that a file of many small
    // leaves is already on the device while the rest of its tasks are made.
    auto block = std::make_shared<std::vector<CopyTask>>(1 + b.larges.size());
    constexpr size_t kSubmitChunk = 1024;
    std::vector<std::shared_ptr<CopyTask>> tasks;
    tasks.reserve(std::min(block->size(), kSubmitChunk));
    auto submit = [&] {
      if (tasks.empty()) return;
      transfers_.submit_copies(ticket->id_, std::move(tasks));
      tasks.clear();
      tasks.reserve(kSubmitChunk);
    };
    auto meta = std::shared_ptr<CopyTask>(block, block->data());
    meta->ticket = ticket->id_;
    meta->shard_id = b.shard_id;
    meta->source.host_ptr = b.meta.get();
    meta->source.host_size = b.meta_size;
    meta->source.host_keep = b.meta;
    meta->length = b.meta_size;
    meta->dst_offset = pad;
    meta->segment_id = seg.id;
    meta->final_for_segment = b.larges.empty();
    tasks.push_back(std::move(meta));
    uint64_t dst = pad + b.meta_size;
    for (size_t k = 0; k < b.larges.size(); ++k) {
      auto t = std::shared_ptr<CopyTask>(block, block->data() + 1 + k);
      t->ticket = ticket->id_;
      t->shard_id = b.shard_id;
      t->source.region = b.larges[k].region;
      t->source.host_blob = b.larges[k].blob;
      t->length = b.larges[k].size;
      t->segment_id = seg.id;
      t->dst_offset = dst;
      t->final_for_segment = k + 1 == b.larges.size();
      dst += b.larges[k].size;
      tasks.push_back(std::move(t));
      if (tasks.size() == kSubmitChunk) submit();
    }
    tr.mark("reserve+register+tasks");
    submit();
    tr.mark("submit");
    total += b.payload;
  }
  ticket->payload_bytes_ = total;

  const double dt = since(t0);
  std::lock_guard lk(mu_);
  ++counters_.captures;
  counters_.bytes_captured += total;
  counters_.capture_seconds += dt;
  counters_.last_capture_seconds = dt;
  return ticket;
}

// Streamer thread: reserves each streamed segment in capture order (blocking
// on pool backpressure, i.e. on the flush draining earlier segments),
// attaches it to its file and submits its copies.
void Engine::streamer_loop() {
  detail::bind_thread_to_node(pool_.numa_node());
  for (;;) {
    StreamJob j;
    {
      std::unique_lock sl(stream_mu_);
      stream_cv_.wait(sl, [&] { return stream_stop_ || !stream_queue_.empty(); });
      if (stream_queue_.empty()) return;
      j = std::move(stream_queue_.front());
      stream_queue_.pop_front();
      stream_busy_ = true;
    }
    bool skip;
    {
      std::lock_guard tl(j.ticket->mu_);
      skip = !j.ticket->stream_error_.empty();
    }
    std::string err;
    if (!skip) {
      try {
        const bool align = j.length >= kAlignMin && j.length + kRingAlign <= pool_.capacity();
        const Segment seg = pool_.reserve(j.length + (align ? kRingAlign - 1 : 0), j.ticket->id_);
        const uint64_t pad = align ? aligned_pad(pool_.segment_data(seg), j.meta_size, j.payload_offset) : 0;
        flush_.attach_segment(j.file_id, seg.id, j.payload_offset, pad, j.length);
        for (auto& t : j.tasks) {
          t->segment_id = seg.id;
          t->dst_offset += pad;
        }
        transfers_.submit_copies(j.ticket->id_, std::move(j.tasks));
      } catch (const std::exception& e) {
        err = e.what();
      }
    }
    if (!err.empty()) {
      // Give up on the rest of this capture: its files end Abandoned once
      // the segments already attached drain.
      std::vector<uint64_t> ids;
      {
        std::lock_guard tl(j.ticket->mu_);
        j.ticket->stream_error_ = err;
        j.ticket->failed_ = true;
        if (j.ticket->failure_reason_.empty()) j.ticket->failure_reason_ = "streaming capture: " + err;
        for (const auto& f : j.ticket->files_) ids.push_back(f.flush_file_id);
      }
      for (uint64_t id : ids) flush_.truncate_stream(id);
    }
    {
      std::lock_guard tl(j.ticket->mu_);
      --j.ticket->streams_pending_;
    }
    j.ticket->done_cv_.notify_all();
    {
      std::lock_guard sl(stream_mu_);
      stream_busy_ = false;
    }
    stream_cv_.notify_all();
  }
}

void Engine::wait_streamed(const std::shared_ptr<CaptureTicket>& ticket) {
  std::unique_lock tl(ticket->mu_);
  ticket->done_cv_.wait(tl, [&] { return ticket->streams_pending_ == 0; });
  if (!ticket->stream_error_.empty()) throw Error("streaming capture failed: " + ticket->stream_error_);
}

void Engine::update_barrier(const std::shared_ptr<CaptureTicket>& ticket) {
  detail::NvtxRange range("lzckpt.fence.host");
  const auto t0 = std::chrono::steady_clock::now();
  auto record = [&] {
    const double dt = since(t0);
    std::lock_guard lk(mu_);
    counters_.barrier_seconds += dt;
    counters_.last_barrier_seconds = dt;
  };
  try {
    wait_streamed(ticket);
    transfers_.wait_pending(ticket->id_);
    wait_relay_reads(ticket);
  } catch (...) {
    record();
    throw;
  }
  {
    std::lock_guard tl(ticket->mu_);
    ticket->barrier_passed_ = true;
  }
  record();
}

void Engine::update_barrier_on_stream(const std::shared_ptr<CaptureTicket>& ticket, void* cuda_stream) {
  detail::NvtxRange range("lzckpt.fence.device");
  const auto t0 = std::chrono::steady_clock::now();
  wait_streamed(ticket);  // streamed segments must all be on the device first
  // the helper's reads of delegated leaves are not on this process's streams:
  // the host waits for them (normally long done by the optimizer step)
  {
    std::unique_lock tl(ticket->mu_);
    ticket->done_cv_.wait(tl, [&] { return ticket->relay_reads_pending_ == 0; });
  }
  if (!transfers_.fence_on_stream(ticket->id_, cuda_stream)) {
    update_barrier(ticket);  // paced channel: copies are host-driven
    return;
  }
  {
    std::lock_guard tl(ticket->mu_);
    ticket->barrier_passed_ = true;
  }
  const double dt = since(t0);
  std::lock_guard lk(mu_);
  counters_.barrier_seconds += dt;
  counters_.last_barrier_seconds = dt;
}

void Engine::wait_persisted(const std::shared_ptr<CaptureTicket>& ticket) {
  std::unique_lock tl(ticket->mu_);
  ticket->done_cv_.wait(tl, [&] { return ticket->failed_ || ticket->files_done_ == ticket->files_.size(); });
  if (ticket->torn_) throw TornSnapshot(ticket->failure_reason_);
  if (ticket->failed_) throw Error(ticket->failure_reason_);
}

void Engine::drain() {
  {
    std::unique_lock sl(stream_mu_);
    stream_cv_.wait(sl, [&] { return stream_queue_.empty() && !stream_busy_; });
  }
  transfers_.drain();
  flush_.drain();
}

void Engine::on_file_done(const std::shared_ptr<CaptureTicket>& ticket, FlushFileState state) {
  {
    std::lock_guard tl(ticket->mu_);
    ++ticket->files_done_;
    if (state == FlushFileState::Abandoned && !ticket->failed_) {
      ticket->failed_ = true;
      if (ticket->failure_reason_.empty()) {
        ticket->failure_reason_ = "a shard file flush was abandoned before its header was written";
      }
    }
  }
  ticket->done_cv_.notify_all();
}

void Engine::on_torn(uint64_t ticket_id) {
  std::shared_ptr<CaptureTicket> ticket;
  {
    std::lock_guard lk(mu_);
    auto it = tickets_.find(ticket_id);
    if (it != tickets_.end()) ticket = it->second.lock();
  }
  if (!ticket) return;
  std::vector<uint64_t> ids;
  {
    std::lock_guard tl(ticket->mu_);
    ticket->torn_ = true;
    ticket->failed_ = true;
    ticket->failure_reason_ =
        "a source region changed while step " + std::to_string(ticket->step_) + " copies were pending";
    for (const auto& f : ticket->files_) ids.push_back(f.flush_file_id);
  }
  for (uint64_t id : ids) flush_.abandon(id);  // these files never gain a header
  ticket->done_cv_.notify_all();
}

TicketStatus Engine::ticket_status(const CaptureTicket& t) const {
  if (t.failed_) return TicketStatus::Failed;
  if (t.files_done_ == t.files_.size()) return TicketStatus::Persisted;
  if (t.relay_reads_pending_ > 0) return TicketStatus::InFlight;
  if (t.streamed_) {
    return t.streams_pending_ == 0 && transfers_.ticket_complete(t.id_) ? TicketStatus::HostResident
                                                                         : TicketStatus::InFlight;
  }
  for (const auto& f : t.files_) {
    try {
      if (pool_.segment_state(f.segment_id) == SegmentState::Reserved) return TicketStatus::InFlight;
    } catch (const IllegalTransition&) {
      // already released; the file callback is on its way
    }
  }
  return TicketStatus::HostResident;
}

std::vector<CheckpointFileHeader> Engine::ticket_headers(const std::shared_ptr<CaptureTicket>& ticket) const {
  std::vector<uint64_t> ids;
  {
    std::lock_guard tl(ticket->mu_);
    for (const auto& f : ticket->files_) ids.push_back(f.flush_file_id);
  }
  std::vector<CheckpointFileHeader> out;
  for (uint64_t id : ids) out.push_back(const_cast<FlushPipeline&>(flush_).file_header(id));
  return out;
}

void Engine::wait_relay_reads(const std::shared_ptr<CaptureTicket>& ticket) {
  std::unique_lock tl(ticket->mu_);
  ticket->done_cv_.wait(tl, [&] { return ticket->relay_reads_pending_ == 0; });
  if (ticket->torn_) throw TornSnapshot(ticket->failure_reason_);
  if (ticket->failed_) throw Error(ticket->failure_reason_);
}

// Hands one file's delegated leaves to the helper. Torn rule as for local
// copies: a leaf whose version moved before the helper finished reading it
// tears the ticket (reference transfer_engine.cpp:146-154).
void Engine::relay_submit(const std::shared_ptr<CaptureTicket>& ticket, const std::filesystem::path& path,
                          uint64_t file_id, const std::vector<std::shared_ptr<DeviceRegion>>& regions,
                          const std::vector<uint64_t>& sizes, const std::vector<uint64_t>& file_offsets,
                          void* producer_stream, bool ordered) {
  {
    std::lock_guard tl(ticket->mu_);
    ++ticket->relay_reads_pending_;
  }
  std::vector<uint64_t> versions(regions.size());
  for (size_t i = 0; i < regions.size(); ++i) versions[i] = regions[i]->version();
  std::weak_ptr<CaptureTicket> weak = ticket;
  const uint64_t ticket_id = ticket->id_;
  lzk_event* ev = nullptr;
  lzk_ipc_handle evh{};
  // READ_DONE (or a failure): settle the ticket's relay part
  auto on_read = [this, weak, ticket_id, regions, versions](bool ok, const std::string& err) {
    bool torn = false;
    for (size_t i = 0; i < regions.size(); ++i) torn = torn || regions[i]->version() != versions[i];
    auto t = weak.lock();
    if (!t) return;
    if (torn && ok) on_torn(ticket_id);
    {
      std::lock_guard tl(t->mu_);
      --t->relay_reads_pending_;
      if (!ok && !t->failed_) {
        t->failed_ = true;
        if (t->failure_reason_.empty()) t->failure_reason_ = "uplink relay: " + err;
      }
    }
    t->done_cv_.notify_all();
  };
  try {
    std::vector<detail::RelayEntry> entries(regions.size());
    uint64_t bytes = 0;
    for (size_t i = 0; i < regions.size(); ++i) {
      // exported at every capture: an allocation freed and re-made at the
      // same address gets a new handle, which a cache keyed by address
      // would miss (the helper would then read the old allocation)
      uint64_t off = 0;
      ck(lzk_ipc_export_mem(regions[i]->device(), regions[i]->device_ptr(), &entries[i].mem, &off),
         "relay: export a leaf");
      entries[i].src_offset = off;
      entries[i].length = sizes[i];
      entries[i].file_offset = file_offsets[i];
      bytes += sizes[i];
    }
    // producer ordering across processes: an interprocess event on the trainer's stream
    if (ordered) {
      {
        std::lock_guard lk(relay_mu_);
        if (!relay_events_.empty()) {
          std::tie(ev, evh) = relay_events_.back();
          relay_events_.pop_back();
        }
      }
      if (!ev) ck(lzk_ipc_event_create(transfers_.device(), &ev, &evh), "relay: producer event");
      ck(lzk_event_record_raw(ev, producer_stream), "relay: record on the producer stream");
    }
    uint32_t flags = 0;
    if (!config_.flush.discard) flags |= detail::kRelayHash;
    if (!config_.flush.discard && !config_.flush.hash_only) flags |= detail::kRelayWrite;
    if (!config_.flush.discard && config_.flush.fsync_on_finalize) flags |= detail::kRelayFsync;
    lzk_event* used = ev;
    auto read_done = [this, on_read, used, evh](bool ok, const std::string& err) {
      if (used) {
        std::lock_guard lk(relay_mu_);
        relay_events_.emplace_back(used, evh);  // the helper has consumed its wait
      }
      on_read(ok, err);
    };
    auto persisted = [this, file_id](bool ok, const std::string&, const std::vector<uint64_t>& sums) {
      flush_.complete_external(file_id, ok, sums);
    };
    relay_client_->submit(path, flags, ev ? &evh : nullptr, entries, read_done, persisted);
    std::lock_guard lk(relay_mu_);
    relay_delegated_ += bytes;
  } catch (const std::exception& e) {
    // The helper is unreachable: the ticket fails (its own copies still run,
    // so the pool drains) and the file ends without a header.
    if (ev) {
      std::lock_guard lk(relay_mu_);
      relay_events_.emplace_back(ev, evh);
    }
    on_read(false, e.what());
    flush_.complete_external(file_id, false, {});
  }
}

void Engine::set_relay(const std::string& peer_socket, double share) {
  if (share < 0 || share >= 1) throw ConfigError("relay share must be in [0, 1)");
  std::unique_ptr<detail::RelayClient> fresh;
  bool need = false;
  {
    std::lock_guard lk(relay_mu_);
    need = share > 0 && !relay_client_;
  }
  if (need) fresh = std::make_unique<detail::RelayClient>(peer_socket);  // connects (may wait for the helper)
  std::lock_guard lk(relay_mu_);
  if (fresh) relay_client_ = std::move(fresh);
  relay_share_ = share;
}

Engine::RelayStats Engine::relay_stats() const {
  RelayStats s;
  {
    std::lock_guard lk(relay_mu_);
    s.delegated_bytes = relay_delegated_;
  }
  if (relay_server_) {
    s.served_bytes = relay_server_->bytes_relayed();
    s.served_requests = relay_server_->requests();
  }
  return s;
}

Engine::Counters Engine::counters() const {
  std::lock_guard lk(mu_);
  return counters_;
}

std::vector<std::byte> read_entry(const std::filesystem::path& file, const CheckpointFileHeader& header,
                                  std::string_view key) {
  const HeaderEntry* e = header.find(key);
  if (!e) throw FormatError(file.string() + ": no entry named '" + std::string(key) + "'");
  const int fd = ::open(file.c_str(), O_RDONLY | O_CLOEXEC);
  if (fd < 0) throw IoError("cannot open " + file.string());
  std::vector<std::byte> out(e->length);
  uint64_t got = 0;
  while (got < e->length) {
    ssize_t r = ::pread(fd, out.data() + got, e->length - got, off_t(e->offset + got));
    if (r < 0 && errno == EINTR) continue;
    if (r <= 0) break;
    got += uint64_t(r);
  }
  ::close(fd);
  if (got != e->length) {
    throw TruncatedFile(file.string() + ": short read for entry '" + std::string(key) + "'");
  }
  return out;
}

namespace {

// Header + exact-extent check (reference read_header + validate_entries
// length rule, format.cpp:173-214) and the parsed __meta__ leaf manifest.
std::vector<LeafManifestEntry> open_shard(const std::filesystem::path& path, CheckpointFileHeader& h) {
  h = read_header(path);
  std::error_code ec;
  const uint64_t size = std::filesystem::file_size(path, ec);
  if (ec) throw IoError("cannot stat " + path.string());
  if (size != h.payload_end()) {
    throw TruncatedFile("file length " + std::to_string(size) + " does not match declared extent " +
                        std::to_string(h.payload_end()));
  }
  auto meta = read_entry(path, h, StateTree::kMetaKey);
  if (fnv64(meta.data(), meta.size()) != h.find(StateTree::kMetaKey)->checksum) {
    // corrupt metadata: report every bad entry, as the reference's
    // validate-before-parse order does (engine.cpp:360-367)
    auto bad = validate_entries(path, h);
    std::string keys;
    for (const auto& k : bad) keys += (keys.empty() ? "" : ", ") + k;
    throw ChecksumMismatch(path.string() + ": corrupt entries: " + keys);
  }
  return parse_leaf_manifest(meta);
}

void throw_bad(const std::filesystem::path& path, const std::vector<std::string>& bad) {
  if (bad.empty()) return;
  std::string keys;
  for (const auto& k : bad) keys += (keys.empty() ? "" : ", ") + k;
  throw ChecksumMismatch(path.string() + ": corrupt entries: " + keys);
}

}  // namespace

namespace {

// One validated shard file into `tree`: region leaves DMA'd into the
// same-path, same-size regions of `into` when present, else fresh regions;
// blobs and inline leaves from host bytes. Reads each byte once.
void restore_one(const std::filesystem::path& path, StateTree& tree, const StateTree* into, int dev,
                 FileStreamer& streamer) {
  detail::NvtxRange range("lzckpt.restore.file");
  PhaseTrace tr("restore_one");
  CheckpointFileHeader h;
  auto leaves = open_shard(path, h);
  tr.mark("open_shard");
  std::vector<EntrySink> sinks(h.entries.size());
  std::vector<std::vector<std::byte>> hostbufs(h.entries.size());
  std::vector<std::shared_ptr<DeviceRegion>> regions(leaves.size());
  auto reuse = [&](const LeafManifestEntry& l) -> std::shared_ptr<DeviceRegion> {
    if (into && into->has(l.path)) {
      try {
        auto r = into->region_at(l.path);
        if (r->size() == l.size && r->device() == dev) return r;
      } catch (const Error&) {
        // a blob at that path: a fresh region instead
      }
    }
    return nullptr;
  };
  // Fresh regions are carved from one device block per file (one allocation
  // instead of one per tensor); the block lives as long as any of them.
  uint64_t fresh = 0;
  for (const auto& l : leaves) {
    if (l.is_region && !reuse(l)) fresh += (l.size + 255) & ~uint64_t(255);
  }
  std::shared_ptr<void> block;
  if (fresh) {
    void* p = nullptr;
    ck(lzk_dev_alloc(dev, fresh, &p), "restore: device allocation");
    block = std::shared_ptr<void>(p, [dev](void* q) { lzk_dev_free(dev, q); });
  }
  uint64_t carved = 0;
  auto region_for = [&](const LeafManifestEntry& l) {
    if (auto r = reuse(l)) {
      r->bump_version();  // contents are being replaced
      return r;
    }
    void* p = static_cast<std::byte*>(block.get()) + carved;
    carved += (l.size + 255) & ~uint64_t(255);
    return DeviceRegion::wrap(p, l.size, dev, block);
  };
  for (size_t e = 0; e < h.entries.size(); ++e) {
    if (h.entries[e].key == StateTree::kMetaKey) {
      hostbufs[e].resize(h.entries[e].length);
      sinks[e].host = &hostbufs[e];
    }
  }
  for (size_t i = 0; i < leaves.size(); ++i) {
    const auto& l = leaves[i];
    if (l.inlined) {
      if (l.inline_bytes.size() != l.size) throw FormatError(path.string() + ": leaf '" + l.path + "' size mismatch");
      continue;
    }
    const HeaderEntry* he = h.find(l.path);
    if (!he) throw FormatError(path.string() + ": no entry named '" + l.path + "'");
    if (he->length != l.size) throw FormatError(path.string() + ": leaf '" + l.path + "' size mismatch");
    const size_t e = size_t(he - h.entries.data());
    if (l.is_region) {
      regions[i] = region_for(l);
      sinks[e].device = regions[i]->device_ptr();
    } else {
      hostbufs[e].resize(l.size);
      sinks[e].host = &hostbufs[e];
    }
  }
  tr.mark("regions");
  bool live = false;  // does the stream write into caller-owned regions?
  for (const auto& l : leaves) live = live || (!l.inlined && l.is_region && reuse(l));
  if (live) {
    // caller-owned regions (e.g. wrapped torch tensors) are written only
    // after every entry checksum has passed: a corrupt file must leave them
    // untouched (restore_into's rule)
    throw_bad(path, streamer.run(path, h, std::vector<EntrySink>(h.entries.size())));
    tr.mark("validate");
  }
  throw_bad(path, streamer.run(path, h, sinks));
  tr.mark("stream");
  std::vector<lzk_copy_desc> inl;
  Pinned stage;
  uint64_t inline_total = 0;
  for (const auto& l : leaves) inline_total += (l.inlined && l.is_region) ? l.size : 0;
  stage.ensure(inline_total);
  uint64_t so = 0;
  for (size_t i = 0; i < leaves.size(); ++i) {
    auto& l = leaves[i];
    if (l.inlined) {
      if (l.is_region) {
        regions[i] = region_for(l);
        if (l.size) {
          std::memcpy(stage.p + so, l.inline_bytes.data(), l.size);
          inl.push_back({reinterpret_cast<uint64_t>(stage.p + so), reinterpret_cast<uint64_t>(regions[i]->device_ptr()),
                         l.size});
          so += l.size;
        }
        tree.set_region(l.path, regions[i]);
      } else {
        tree.set_blob(l.path, std::move(l.inline_bytes));
      }
    } else if (l.is_region) {
      tree.set_region(l.path, regions[i]);
    } else {
      tree.set_blob(l.path, std::move(hostbufs[size_t(h.find(l.path) - h.entries.data())]));
    }
  }
  if (!inl.empty()) {
    lzk_stream* s = nullptr;
    ck(lzk_stream_create(dev, 0, &s), "restore stream");
    int rc = lzk_scatter_h2d(s, inl.data(), uint32_t(inl.size()), 0);
    if (rc == LZK_OK) rc = lzk_stream_sync(s);
    lzk_stream_destroy(s);
    ck(rc, "restore inline leaves");
  }
  tr.mark("inline");
}

}  // namespace

StateTree Engine::restore(const ManifestStore& manifest, uint64_t step) const {
  const auto files = manifest.files_for(step);  // NotCommitted
  const std::string prefix = step_dirname(step) + "/" + rank_dirname(rank_) + "/";
  auto streamer = FileStreamer::acquire(transfers_.device());
  StateTree tree;
  for (const auto& rec : files) {
    if (rec.relative_path.rfind(prefix, 0) != 0) continue;
    restore_one(config_.checkpoint_root / rec.relative_path, tree, nullptr, transfers_.device(), *streamer);
  }
  return tree;
}

StateTree Engine::restore_file(const std::filesystem::path& path, const StateTree* into) const {
  auto streamer = FileStreamer::acquire(transfers_.device());
  StateTree tree;
  restore_one(path, tree, into, transfers_.device(), *streamer);
  return tree;
}

void Engine::restore_into(const ManifestStore& manifest, uint64_t step, StateTree& tree) const {
  const auto files = manifest.files_for(step);
  const std::string prefix = step_dirname(step) + "/" + rank_dirname(rank_) + "/";
  const int dev = transfers_.device();
  auto streamer = FileStreamer::acquire(dev);
  struct Plan {
    std::filesystem::path path;
    CheckpointFileHeader h;
    std::vector<LeafManifestEntry> leaves;
  };
  std::vector<Plan> plans;
  // pass 1: every file's structure and checksums, before any live region is touched
  for (const auto& rec : files) {
    if (rec.relative_path.rfind(prefix, 0) != 0) continue;
    Plan p;
    p.path = config_.checkpoint_root / rec.relative_path;
    p.leaves = open_shard(p.path, p.h);
    for (const auto& l : p.leaves) {
      if (l.is_region) {
        auto r = tree.region_at(l.path);
        if (r->size() != l.size) throw FormatError("restore_into: '" + l.path + "' size mismatch");
        if (r->device() != dev) throw ConfigError("restore_into: '" + l.path + "' on another device");
      }
      if (!l.inlined && !p.h.find(l.path)) throw FormatError(p.path.string() + ": no entry named '" + l.path + "'");
    }
    throw_bad(p.path, streamer->run(p.path, p.h, std::vector<EntrySink>(p.h.entries.size())));
    plans.push_back(std::move(p));
  }
  // pass 2: DMA into the live regions (blobs are host state, left to restore())
  for (auto& p : plans) {
    std::vector<EntrySink> sinks(p.h.entries.size());
    std::vector<std::shared_ptr<DeviceRegion>> touched;
    std::vector<lzk_copy_desc> inl;
    Pinned stage;
    uint64_t inline_total = 0;
    for (const auto& l : p.leaves) inline_total += (l.inlined && l.is_region) ? l.size : 0;
    stage.ensure(inline_total);
    uint64_t so = 0;
    for (const auto& l : p.leaves) {
      if (!l.is_region) continue;
      auto r = tree.region_at(l.path);
      r->bump_version();  // an in-flight capture of this region would be torn
      if (l.inlined) {
        if (l.size) {
          std::memcpy(stage.p + so, l.inline_bytes.data(), l.size);
          inl.push_back({reinterpret_cast<uint64_t>(stage.p + so), reinterpret_cast<uint64_t>(r->device_ptr()), l.size});
          so += l.size;
        }
      } else {
        sinks[size_t(p.h.find(l.path) - p.h.entries.data())].device = r->device_ptr();
      }
      touched.push_back(std::move(r));
    }
    throw_bad(p.path, streamer->run(p.path, p.h, sinks));
    if (!inl.empty()) {
      lzk_stream* s = nullptr;
      ck(lzk_stream_create(dev, 0, &s), "restore stream");
      int rc = lzk_scatter_h2d(s, inl.data(), uint32_t(inl.size()), 0);
      if (rc == LZK_OK) rc = lzk_stream_sync(s);
      lzk_stream_destroy(s);
      ck(rc, "restore inline leaves");
    }
  }
}

}  // namespace lzckpt
