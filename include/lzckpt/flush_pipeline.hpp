// Host-to-storage writer for one rank (streaming flush, header last).
//
// Public contract is the reference's (proj/core/include/lzckpt/flush_pipeline.hpp:38-120,
// src/flush_pipeline.cpp:50-263): files registered with fixed header offsets,
// payload chunks announced in byte order per segment, per-entry FNV-1a folded
// as bytes stream through, header written last (a file without a valid header
// is incomplete), optional fsync, segment released FIFO, abandon and injected
// mid-flush failure.
//
// Unlike the reference (one worker holding the pipeline mutex across pwrite
// and hashing, flush_pipeline.cpp:139-241, which serializes the copy channel
// behind the disk), enqueue_flush only records the chunk; a pool of worker
// threads pwrites pieces in parallel and hashes different entries in
// parallel, each entry's FNV still folded strictly in byte order.
#pragma once

#include <chrono>
#include <condition_variable>
#include <cstdint>
#include <deque>
#include <filesystem>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "lzckpt/buffer_pool.hpp"
#include "lzckpt/checksum.hpp"
#include "lzckpt/format.hpp"

namespace lzckpt {

struct FlushConfig {
  double storage_bandwidth_Bps = 0;  // <= 0: unthrottled
  bool fsync_on_finalize = true;
  // B200-host extensions
  unsigned threads = 0;              // worker pool size; 0 = auto (<= 8)
  uint64_t write_piece = 32ull << 20; // max bytes per pwrite job
  // Concurrent pwrite jobs; 0 = no limit beyond `threads`. The GPU boxes'
  // virtio disk persists a C2 sample at 3.72 GB/s (median) with 3 writers
  // against 3.35 with 8 (profiles/r02_flush_probe_writers.txt): fewer
  // streams, and still one writer copying into its bounce buffer while
  // another is in the kernel.
  unsigned max_writers = 3;
  // Host-memory tier only: no file is created, nothing is hashed or written;
  // a segment is released as soon as all of its bytes are resident. For
  // measuring the D2H snapshot stage on shards larger than local storage.
  bool discard = false;
  // Verification tier: every entry is hashed exactly as for a real file, the
  // header is built, but nothing is written (full-size parity checks on
  // shards larger than local storage).
  bool hash_only = false;
  // Durable files: the block-aligned interior of every write piece goes to
  // the device with O_DIRECT (through an aligned per-thread bounce buffer;
  // ring addresses are laid out for DMA alignment, not file alignment), the
  // partial edge blocks and the header stay buffered. Falls back to buffered
  // writes where O_DIRECT is unavailable. (B200 hosts' local disk: 4.1-4.3
  // GB/s O_DIRECT vs 2.2 buffered.)
  bool direct_io = true;
};

enum class FlushFileState { Pending, Persisted, Abandoned, Discarded };

class FlushPipeline {
 public:
  using FileDoneCallback = std::function<void(uint64_t file_id, FlushFileState)>;

  FlushPipeline(HostBufferPool& pool, FlushConfig config);
  ~FlushPipeline();
  FlushPipeline(const FlushPipeline&) = delete;
  FlushPipeline& operator=(const FlushPipeline&) = delete;

  // B200 extension `payload_pad`: the payload starts `payload_pad` bytes
  // into the segment (the engine places large leaves 4 KiB-aligned in host
  // memory; the copy engines of some hosts lose ~8 % on misaligned
  // destinations). Chunk offsets stay relative to the segment start.
  uint64_t register_file(std::filesystem::path path, CheckpointFileHeader header,
                         uint64_t segment_id, FileDoneCallback on_done = {}, uint64_t payload_pad = 0);
  // B200 extension — streaming through a pool smaller than the file: the
  // payload arrives in consecutive segments attached as they are reserved;
  // every segment but the last is released as soon as its bytes are written
  // and hashed, the last one after the header (file bytes are unchanged).
  uint64_t register_streamed_file(std::filesystem::path path, CheckpointFileHeader header,
                                  FileDoneCallback on_done = {});
  void attach_segment(uint64_t file_id, uint64_t segment_id, uint64_t payload_offset, uint64_t payload_pad = 0,
                      uint64_t payload_len = 0);  // 0: the whole segment
  // Gives up on the rest of a streamed file (a capture that could not get
  // pool space): it ends Abandoned once the attached segments drain.
  void truncate_stream(uint64_t file_id);
  // B200 extension — uplink relay: payload bytes [payload_offset, end) of a
  // registered file are written into the file by another process (a relay
  // helper). Call right after register_file, before any chunk arrives; the
  // suffix must start at an entry whose hash run holds it alone. Those bytes
  // are neither written nor hashed here; complete_external() accounts them
  // and supplies their entries' checksums (or abandons the file).
  void set_external_suffix(uint64_t file_id, uint64_t payload_offset);
  void complete_external(uint64_t file_id, bool ok, const std::vector<uint64_t>& checksums);
  void enqueue_flush(uint64_t segment_id, uint64_t segment_offset, uint64_t length);
  // B200 extension: several in-order chunks under one lock acquisition.
  void enqueue_flush_spans(const std::vector<ChunkSpan>& spans);
  void abandon(uint64_t file_id);
  void inject_failure_after(uint64_t bytes);
  void drain();
  FlushFileState file_state(uint64_t file_id) const;

  uint64_t bytes_written() const;
  // The file's header as finalized (entry checksums filled in).
  CheckpointFileHeader file_header(uint64_t file_id) const;
  uint64_t files_persisted() const;
  size_t queue_depth() const;

 private:
  // Consecutive entries hashed by one job at a time, strictly in byte order
  // (FNV-1a is sequential per entry); different runs hash in parallel. A run
  // is one large entry or several small ones adding up to >= kRunBytes.
  struct HashRun {
    size_t first = 0, last = 0;  // entries [first, last)
    uint64_t begin = 0, end = 0; // payload-relative byte range
    uint64_t resident = 0;       // bytes [begin, resident) are in the pool
    uint64_t hashed = 0;
    size_t cur = 0;              // entry being folded
    uint64_t state = Fnv64::kOffset;
    bool busy = false;
  };
  // One reserved ring segment holding payload bytes [off, off + len).
  struct SubSeg {
    uint64_t id = 0;
    uint64_t off = 0;
    uint64_t len = 0;
    std::byte* base = nullptr;  // payload byte `off` (segment start + pad)
    uint64_t pad = 0;           // payload offset within the segment
    uint64_t accounted = 0;  // written + starved bytes inside this segment
    bool released = false;
  };
  struct FileRecord {
    std::filesystem::path path;
    CheckpointFileHeader header;
    uint64_t header_size = 0;
    uint64_t expected = 0;
    uint64_t attached = 0;       // payload bytes covered by attached segments
    uint64_t enqueued = 0;       // next in-order chunk offset (= resident end)
    uint64_t write_queued = 0;   // bytes [0, write_queued) handed to writers
    uint64_t starve_from = ~0ull;// injected failure: bytes >= this never reach the disk
    uint64_t accounted = 0;      // written + starved bytes
    uint64_t own_end = ~0ull;    // payload bytes >= own_end arrive externally (relay)
    bool external_done = true;
    uint64_t own_limit() const { return own_end < expected ? own_end : expected; }
    uint32_t jobs = 0;           // outstanding jobs touching this file
    uint32_t writes_inflight = 0;
    std::vector<SubSeg> segs;    // in payload order
    std::vector<uint64_t> entry_begin;  // payload-relative, per entry
    std::vector<HashRun> runs;
    size_t entries_done = 0;
    int fd = -1;
    int dfd = -1;  // O_DIRECT descriptor of the same file (-1: buffered only)
    bool abandoned = false;
    bool finalizing = false;
    bool finalized = false;
    FlushFileState state = FlushFileState::Pending;
    FileDoneCallback on_done;

    size_t seg_index(uint64_t payload_off) const;  // segment holding this byte
  };
  struct Job {
    bool hash = false;
    uint64_t file = 0;
    uint64_t offset = 0;  // write: payload offset
    uint64_t length = 0;  // write: bytes
    size_t run = 0;       // hash: run index
  };
  static constexpr uint64_t kRunBytes = 4ull << 20;

  void queue_writes(uint64_t id, FileRecord& f);
  void enqueue_locked(std::unique_lock<std::mutex>& lk, uint64_t segment_id, uint64_t seg_offset, uint64_t length);
  void account(FileRecord& f, uint64_t from, uint64_t to);
  bool hashed_through(const FileRecord& f, uint64_t end) const;
  uint64_t register_common(std::filesystem::path path, CheckpointFileHeader header, FileDoneCallback on_done,
                           FileRecord& f);
  void worker_loop();
  void run_write(FileRecord& f, const Job& j, const std::byte* src);
  void run_hash(uint64_t file_id, size_t run);
  void maybe_finalize(std::unique_lock<std::mutex>& lk, uint64_t file_id);
  void release_in_order(std::unique_lock<std::mutex>& lk);
  void fail_locked(const std::string& why);

  HostBufferPool& pool_;
  const FlushConfig config_;

  mutable std::mutex mu_;
  std::condition_variable work_cv_;
  std::condition_variable done_cv_;
  std::deque<Job> jobs_;
  std::unordered_map<uint64_t, std::pair<uint64_t, size_t>> seg_to_file_;  // segment -> (file, index)
  std::unordered_map<uint64_t, FileRecord> files_;
  std::deque<std::pair<uint64_t, size_t>> release_order_;  // (file, segment index) in reservation order
  uint64_t next_file_ = 1;
  uint64_t pending_files_ = 0;
  uint32_t callbacks_in_flight_ = 0;
  uint32_t busy_workers_ = 0;
  uint32_t writers_ = 0;  // write jobs running (bounded by config_.max_writers)
  uint64_t bytes_written_ = 0;
  uint64_t files_persisted_ = 0;
  int64_t fail_after_ = -1;
  std::string error_;
  bool stopping_ = false;

  std::mutex pace_mu_;
  std::chrono::steady_clock::time_point pace_point_{};
  std::vector<std::thread> workers_;
};

}  // namespace lzckpt
