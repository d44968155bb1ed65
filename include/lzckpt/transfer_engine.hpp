// Device-to-host snapshot engine for one rank (the hot path).
//
// API mirrors the reference's emulated engine
// (proj/core/include/lzckpt/transfer_engine.hpp:24-134): DeviceRegion with a
// version counter, CopyTask, ThrottledChannel pacing, submit_copies /
// wait_pending / drain, in-order chunk announcements and torn detection.
//
// Underneath it is B200-native:
//  * DeviceRegion owns (or wraps) real HBM;
//  * unpaced submissions are cut into groups on the caller (host metadata
//    only) and issued by a per-engine issuer thread onto a dedicated
//    snapshot stream: tensors below SnapshotOptions::ce_threshold go through
//    ONE multi-tensor gather kernel launch per group (lzk_gather_d2h), larger
//    ones through the copy engines (lzk_ce_copy_d2h); a CUDA event closes
//    every group. capture() therefore never blocks on the device queue;
//  * one completion thread per rank waits on group events in FIFO order and
//    only then decides torn-ness, marks segments Filled and announces chunks,
//    so announcement order and the verdict-before-final-chunk rule are the
//    reference's (transfer_engine.cpp:146-157);
//  * fence_on_stream() is the device-side lazy fence: the trainer's stream
//    waits on the ticket's last event instead of the host blocking.
#pragma once

#include <atomic>
#include <chrono>
#include <cstdlib>
#include <condition_variable>
#include <cstddef>
#include <cstdint>
#include <deque>
#include <functional>
#include <memory>
#include <mutex>
#include <span>
#include <thread>
#include <unordered_map>
#include <vector>

#include "lzckpt/buffer_pool.hpp"
#include "lzk_cuda.h"



namespace lzckpt {

// HBM allocation with the reference's version semantics: every update-phase
// mutation bumps the version; a copy that observes a bump between submit and
// completion is torn.
class DeviceRegion {
 public:
  // device < 0: the calling thread's current CUDA device.
  explicit DeviceRegion(uint64_t size, int device = -1);
  explicit DeviceRegion(std::vector<std::byte> initial, int device = -1);
  // Allocation without the zero fill (restore overwrites every byte).
  struct Uninitialized {};
  DeviceRegion(Uninitialized, uint64_t size, int device = -1);
  ~DeviceRegion();
  DeviceRegion(const DeviceRegion&) = delete;
  DeviceRegion& operator=(const DeviceRegion&) = delete;

  // Non-owning view of memory someone else allocated (e.g. a torch tensor).
  static std::shared_ptr<DeviceRegion> wrap(void* device_ptr, uint64_t size, int device);
  // Same, keeping `owner` (e.g. a block several regions are carved from)
  // alive for as long as the region lives.
  static std::shared_ptr<DeviceRegion> wrap(void* device_ptr, uint64_t size, int device,
                                            std::shared_ptr<void> owner);

  uint64_t size() const { return size_; }
  uint64_t version() const { return version_.load(std::memory_order_acquire); }

  // Staged host-side mutation (D2H -> fn -> H2D), one version bump.
  void mutate(const std::function<void(std::span<std::byte>)>& fn);
  void write(uint64_t offset, std::span<const std::byte> data);
  void read_chunk(uint64_t offset, std::span<std::byte> out) const;
  std::vector<std::byte> clone_bytes() const;

  // B200 extensions
  void* device_ptr() const { return ptr_; }
  int device() const { return device_; }
  // Declares an in-place device-side mutation (e.g. the optimizer step ran on
  // a CUDA stream): same effect on torn detection as mutate().
  void bump_version() { version_.fetch_add(1, std::memory_order_acq_rel); }
  std::mutex& io_mutex() const { return mu_; }

 private:
  struct WrapTag {};
  DeviceRegion(WrapTag, void* ptr, uint64_t size, int device);

  mutable std::mutex mu_;
  void* ptr_ = nullptr;
  uint64_t size_ = 0;
  int device_ = 0;
  bool owned_ = true;
  std::atomic<uint64_t> version_{0};
};

// Bandwidth model for one copy link. bandwidth_Bps <= 0 disables pacing
// (the measured fast path); > 0 paces chunk by chunk, as the reference.
struct ThrottledChannel {
  double bandwidth_Bps = 25e9;
  uint64_t chunk_quantum = 64ull << 20;
};

// B200 extension: how unpaced snapshots are issued on the device.
struct SnapshotOptions {
  int device = -1;                    // -1: current device at construction
  uint64_t ce_threshold = 2ull << 20; // tasks >= this go to the copy engines
  // gather kernel grid: 2 CTAs already saturate the host link in every size
  // class (profiles/r02_ctasweep.jsonl); 4 leave margin and take 2.7 % of the SMs
  uint32_t kernel_ctas = 4;
  uint64_t group_bytes = 256ull << 20; // bytes per completion event (and max DMA size)
  // > 0: the least priority, < 0: the greatest. CUDA's least priority IS the
  // default (0), so the snapshot stream never ranks below an ordinary compute
  // stream; a trainer that wants its kernels scheduled ahead of the gather
  // kernel creates its own stream at a greater (negative) priority.
  int stream_priority = 1;
  bool force_kernel = false;          // every region chunk through the gather kernel
  bool force_copy_engine = false;     // every region chunk through the copy engines
};

enum class CopyState { Queued, Copying, Done, Torn };

struct CopySource {
  std::shared_ptr<DeviceRegion> region;
  std::shared_ptr<const std::vector<std::byte>> host_blob;
  // B200 extension: host bytes in pinned memory kept alive by `host_keep`
  // (the engine's __meta__, whose inline leaves the gather kernel writes in
  // place). A task has exactly one of region / host_blob / host_ptr.
  const std::byte* host_ptr = nullptr;
  uint64_t host_size = 0;
  std::shared_ptr<const void> host_keep;

  bool is_host() const { return host_blob != nullptr || host_ptr != nullptr; }
  const std::byte* host_data() const { return host_blob ? host_blob->data() : host_ptr; }
  uint64_t host_bytes() const { return host_blob ? host_blob->size() : host_size; }
};

struct CopyTask {
  uint64_t ticket = 0;
  uint64_t shard_id = 0;
  CopySource source;
  uint64_t src_offset = 0;
  uint64_t length = 0;
  uint64_t segment_id = 0;
  uint64_t dst_offset = 0;  // within the segment
  uint64_t captured_version = 0;
  bool final_for_segment = false;
  std::atomic<CopyState> state{CopyState::Queued};
  // B200 extension: version observed when the device-side fence was placed;
  // mutations after the fence are stream-ordered behind the copy.
  uint64_t fence_version = 0;
  bool fenced = false;
};

class TransferEngine {
 public:
  using ChunkCallback = std::function<void(uint64_t, uint64_t, uint64_t)>;
  using TornCallback = std::function<void(const CopyTask&)>;

  TransferEngine(HostBufferPool& pool, ThrottledChannel channel);
  TransferEngine(HostBufferPool& pool, ThrottledChannel channel, SnapshotOptions options);
  ~TransferEngine();
  TransferEngine(const TransferEngine&) = delete;
  TransferEngine& operator=(const TransferEngine&) = delete;

  void set_chunk_callback(ChunkCallback cb) { chunk_cb_ = std::move(cb); }
  // B200 extension: one call per completed device group, its chunks
  // coalesced into contiguous spans (the engine feeds the flush this way;
  // thousands of small tensors become a few notices). When set it replaces
  // the per-chunk callback on the device path; the paced path and the
  // reference's per-chunk contract are unchanged without it.
  using SpanCallback = std::function<void(const std::vector<ChunkSpan>&)>;
  void set_span_callback(SpanCallback cb) { span_cb_ = std::move(cb); }
  void set_torn_callback(TornCallback cb) { torn_cb_ = std::move(cb); }

  // Non-blocking: validates, enqueues the device work, returns.
  void submit_copies(uint64_t ticket, std::vector<std::shared_ptr<CopyTask>> tasks);
  void wait_pending(uint64_t ticket);
  bool ticket_torn(uint64_t ticket) const;
  void drain();

  uint64_t bytes_submitted() const { return bytes_submitted_.load(); }
  uint64_t bytes_delivered() const { return bytes_delivered_.load(); }
  const ThrottledChannel& channel() const { return channel_; }

  // ---- B200 extensions ----
  // Device-side lazy fence: work queued on `cuda_stream` after this call runs
  // after every copy of `ticket`. Returns false when the ticket's copies are
  // not device-issued (paced channel); the caller then waits on the host.
  bool fence_on_stream(uint64_t ticket, void* cuda_stream);
  // Producer ordering (capture on a trainer stream). Records an event on
  // `producer_stream` now (NULL = the legacy default stream); the ticket's
  // device work waits for it, so the snapshot reads what the trainer queued
  // before capture() and never a half-written tensor. `inline_descs` (small
  // leaves gathered straight into their __meta__ slots) then run first on the
  // snapshot stream, and `inline_regions` get the same torn verdict as large
  // leaves (the reference clones them at capture, engine.cpp:138-143; here
  // that read is deferred behind the producer instead of blocking the
  // trainer). Call before the ticket's first submit_copies.
  // `keep` holds the inline descriptors' destinations (the __meta__ buffers)
  // until the gather has completed, even if the capture is abandoned.
  void set_prologue(uint64_t ticket, void* producer_stream, std::vector<lzk_copy_desc> inline_descs,
                    std::vector<std::shared_ptr<DeviceRegion>> inline_regions,
                    std::vector<std::shared_ptr<const void>> keep = {});
  bool ticket_complete(uint64_t ticket) const;
  // Device time of a completed ticket's snapshot (CUDA events on the snapshot
  // stream, first device op -> last completion); < 0 when not measured.
  double ticket_device_ms(uint64_t ticket) const;
  // A capture that submits several files holds its ticket until the last is
  // submitted, so that an early file completing first does not close the
  // ticket's device time. Unheld tickets (direct submit_copies users) close
  // whenever everything submitted so far has completed.
  void hold(uint64_t ticket);
  void seal(uint64_t ticket);
  const SnapshotOptions& options() const { return opts_; }
  // Changes the variant selection for subsequent submissions (device and
  // stream priority are fixed at construction).
  void set_options(const SnapshotOptions& o);
  int device() const { return device_; }
  lzk_stream* stream() const { return stream_; }

  struct Stats {
    uint64_t kernel_launches = 0;  // gather launches issued
    uint64_t kernel_bytes = 0;
    uint64_t ce_copies = 0;
    uint64_t ce_bytes = 0;
    uint64_t blob_bytes = 0;
    uint64_t groups = 0;
  };
  Stats stats() const;

 private:
  struct Piece {
    CopyTask* task = nullptr;  // owned by the ticket's task list until its last group is done
    uint64_t offset = 0;  // within the task
    uint64_t length = 0;
    bool last = false;
  };
  struct Group {
    uint64_t ticket = 0;
    bool paced = false;          // copied chunk by chunk by the completion thread
    std::vector<Piece> pieces;
    std::vector<lzk_copy_desc> kernel;  // gather-kernel descriptors (small tensors)
    std::vector<lzk_copy_desc> dma;     // copy-engine descriptors (large tensors)
    uint32_t kernel_ctas = 0;    // gather grid for this group
    lzk_event* done = nullptr;   // recorded after the group's device work
    bool issue_failed = false;
    bool host_after_device = false;  // host copies read bytes the prologue writes
  };
  struct InlineWatch {
    std::shared_ptr<DeviceRegion> region;
    uint64_t captured = 0;
    uint64_t fence = 0;
    bool fenced = false;
  };
  struct TicketProgress {
    uint64_t expected = 0;
    uint64_t completed = 0;
    uint64_t unissued = 0;       // groups queued but not yet on the device
    bool torn = false;
    bool device_issued = true;
    lzk_event* last_event = nullptr;
    lzk_event* start_event = nullptr;  // recorded before the ticket's first group
    double device_ms = -1;             // first issue -> last completion, on the device
    std::vector<std::shared_ptr<CopyTask>> tasks;  // for fence versions
    // set_prologue: consumed by the issuer before the ticket's first group
    lzk_event* producer = nullptr;
    std::vector<lzk_copy_desc> inline_descs;
    bool prologue = false;                 // the ticket's __meta__ is written on the device
    std::vector<InlineWatch> inline_watch;  // verdict at the first completed group
    std::vector<std::shared_ptr<const void>> inline_keep;  // until the first group completes
    // LZCKPT_TRACE: host-side timeline of the ticket's device path
    std::chrono::steady_clock::time_point t_submit{}, t_first_issue{}, t_last_issue{}, t_last_sync{};
    bool held = false;                 // hold()/seal(): more files may still be submitted
    lzk_event* final_event = nullptr;  // the last completed group's event, until device_ms is taken
  };

  void issuer_loop();
  void worker_loop();
  void run_device_group(Group& g);
  void run_paced_group(Group& g);
  void build_groups(const std::vector<std::shared_ptr<CopyTask>>& tasks, std::deque<Group>& out);
  void issue(Group& g);
  void finalize_device_time(uint64_t ticket, TicketProgress& tp);
  lzk_event* take_event();
  void give_event(lzk_event* e);

  HostBufferPool& pool_;
  const bool trace_ = std::getenv("LZCKPT_TRACE") != nullptr;
  const ThrottledChannel channel_;
  SnapshotOptions opts_;
  int device_ = 0;
  lzk_stream* stream_ = nullptr;
  ChunkCallback chunk_cb_;
  SpanCallback span_cb_;
  TornCallback torn_cb_;

  std::mutex opts_mu_;
  mutable std::mutex mu_;
  std::condition_variable issue_cv_;
  std::condition_variable issued_cv_;
  std::condition_variable work_cv_;
  std::condition_variable progress_cv_;
  std::deque<Group> issue_queue_;  // built on the caller, issued by issuer_
  std::deque<Group> queue_;        // issued, awaiting completion on worker_
  std::unordered_map<uint64_t, TicketProgress> tickets_;
  std::vector<lzk_event*> free_events_;
  uint64_t in_flight_ = 0;
  bool issuing_ = false;
  bool stopping_ = false;
  bool issuer_done_ = false;
  Stats stats_;

  std::atomic<uint64_t> bytes_submitted_{0};
  std::atomic<uint64_t> bytes_delivered_{0};
  std::chrono::steady_clock::time_point pace_point_{};
  std::thread issuer_;
  std::thread worker_;
};

}  // namespace lzckpt
