// Uplink relay between the ranks of one node (B200 extension; no reference
// counterpart — the reference has one emulated link per rank).
//
// On hosts where several GPUs share one PCIe uplink, the slowest rank sets
// every checkpoint's time. Measured (profiles/r02_relay_*): a
// D2H DMA issued on GPU B with GPU A's memory as source does NOT use B's
// link, but B's copy engines pulling A's memory into B's HBM (D2D over
// NVLink) and then DMAing it to host do, at the full DMA rate; so does an SM
// kernel on B reading A's HBM and storing to host, at a lower rate and with
// SMs held. The relay runs in the HELPER's own process:
//
//   owner  capture() keeps a suffix of each shard file's large leaves out of
//          its own D2H and sends them as a request: CUDA IPC handles of the
//          leaves' allocations, the shard file and the leaves' file offsets,
//          and an interprocess event recorded on the producer stream;
//   helper waits for that event on its relay streams, pulls the leaves
//          from the owner's HBM through IPC into HBM staging (D2D), DMAs each
//          staged chunk into pinned staging on its own link (or, SM route,
//          gathers straight from the IPC source), reports READ_DONE (the owner's lazy fence
//          needs it), then pwrites the bytes at their offsets in the owner's
//          file, optionally hashes them (device FNV over the IPC source) and
//          fsyncs, and reports PERSISTED with the entry checksums;
//   owner  its flush treats the suffix as external bytes: accounted, not
//          written, checksums taken from the reply; the header still goes
//          last, so the file format and the header-last rule are unchanged.
//
// Transport: a Unix stream socket per helper, length-prefixed frames.
#pragma once

#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <cstdint>
#include <filesystem>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <string>
#include <thread>
#include <vector>

#include "lzk_cuda.h"

namespace lzckpt::detail {

// One delegated leaf.
struct RelayEntry {
  lzk_ipc_handle mem;        // the owner's allocation holding the leaf
  uint64_t src_offset = 0;   // leaf offset inside that allocation
  uint64_t length = 0;
  uint64_t file_offset = 0;  // absolute offset of the leaf in the shard file
};

enum RelayFlags : uint32_t {
  kRelayWrite = 1,   // pwrite the bytes into the file
  kRelayHash = 2,    // return each entry's FNV-1a-64
  kRelayFsync = 4,   // fsync the file before PERSISTED
};

class RelayServer {
 public:
  // Serves owners on `socket_path` with the gather kernel on `device`
  // (`ctas` CTAs) through `staging_bytes` of pinned staging.
  // copy_engines: pull each chunk over NVLink into HBM staging with a D2D
  // copy, then DMA it to host over this GPU's link (no SM time taken from
  // the helper's training); false: the gather kernel reads the owner's HBM
  // directly and stores to host (SM path).
  RelayServer(int device, std::string socket_path, uint64_t staging_bytes, uint32_t ctas, bool copy_engines = true);
  ~RelayServer();
  RelayServer(const RelayServer&) = delete;
  RelayServer& operator=(const RelayServer&) = delete;

  const std::string& path() const { return path_; }
  uint64_t bytes_relayed() const;
  uint64_t requests() const;

 private:
  struct Request;
  void accept_loop();
  void serve(int fd);
  void handle(int fd, Request& r);

  const int device_;
  const std::string path_;
  const uint64_t chunk_;
  const uint32_t ctas_;
  const bool copy_engines_;
  int listen_fd_ = -1;
  lzk_stream* stream_ = nullptr;       // gathers / D2H
  lzk_stream* pull_stream_ = nullptr;  // copy-engine route: D2D pulls over NVLink
  std::vector<void*> dev_stage_;       // copy-engine route: HBM staging chunks
  std::vector<lzk_event*> pulled_;
  lzk_stream* hash_stream_ = nullptr;  // entry checksums, beside the gathers
  std::vector<std::byte*> staging_;  // pinned, mapped chunks
  std::vector<lzk_event*> chunk_done_;
  uint64_t* digests_ = nullptr;      // pinned, mapped: per-entry FNV results
  uint32_t digest_cap_ = 0;
  std::map<std::string, lzk_event*> events_;  // opened producer events by handle bytes
  static constexpr size_t kMaxOpen = 4096;    // owners' allocations kept mapped
  std::set<std::string> opened_;

  const bool trace_ = std::getenv("LZCKPT_TRACE") != nullptr;  // per-request timing on stderr
  std::chrono::steady_clock::time_point last_done_{};
  mutable std::mutex mu_;  // one request at a time (the staging is shared)
  uint64_t bytes_ = 0;
  uint64_t requests_ = 0;
  bool stop_ = false;
  std::thread acceptor_;
  std::vector<std::thread> conns_;
  std::vector<int> conn_fds_;
};

class RelayClient {
 public:
  explicit RelayClient(const std::string& socket_path);
  ~RelayClient();
  RelayClient(const RelayClient&) = delete;
  RelayClient& operator=(const RelayClient&) = delete;

  using ReadDone = std::function<void(bool ok, const std::string& error)>;
  using Persisted = std::function<void(bool ok, const std::string& error, const std::vector<uint64_t>& checksums)>;
  // Sends one request; the callbacks run on the client's reader thread,
  // READ_DONE before PERSISTED. `producer` may be null (no ordering).
  void submit(const std::filesystem::path& file, uint32_t flags, const lzk_ipc_handle* producer,
              const std::vector<RelayEntry>& entries, ReadDone on_read, Persisted on_persisted);
  bool connected() const;

 private:
  void reader_loop();
  void fail_all(const std::string& why);

  int fd_ = -1;
  mutable std::mutex mu_;
  std::mutex send_mu_;
  uint64_t next_ = 1;
  struct Pending {
    ReadDone on_read;
    Persisted on_persisted;
    bool read = false;
    std::chrono::steady_clock::time_point sent{};
  };
  const bool trace_ = std::getenv("LZCKPT_TRACE") != nullptr;
  std::map<uint64_t, Pending> pending_;
  bool broken_ = false;
  std::thread reader_;
};

}  // namespace lzckpt::detail
