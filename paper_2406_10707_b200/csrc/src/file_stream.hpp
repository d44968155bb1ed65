// Internal to liblzckpt_b200.so: streaming a checkpoint file back through
// the GPU (restore, commit-time validation) and small host utilities shared
// by engine.cpp and consolidation.cpp. Not part of the public headers.
#pragma once

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <memory>
#include <string>
#include <vector>

#include "lzckpt/format.hpp"
#include "lzk_cuda.h"

namespace lzckpt::detail {

void ck(int rc, const char* what);  // DeviceError on a failed lzk_* call

inline double since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// LZCKPT_TRACE=1: per-phase timing on stderr (host-overhead tuning).
struct PhaseTrace {
  explicit PhaseTrace(const char* what = "capture") : what(what) {}
  const char* what;
  bool on = std::getenv("LZCKPT_TRACE") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  std::string line;
  void mark(const char* name) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    line += std::string(" ") + name + "=" + std::to_string(std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
  ~PhaseTrace() {
    if (on) std::fprintf(stderr, "[lzckpt %s ms]%s\n", what, line.c_str());
  }
};

// NVTX range for the lifetime of the object (a no-op without a profiler).
struct NvtxRange {
  explicit NvtxRange(const char* name) { lzk_range_push(name); }
  ~NvtxRange() { lzk_range_pop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// Where one entry's bytes go while a file streams back.
struct EntrySink {
  void* device = nullptr;                 // region memory (device address), or
  std::vector<std::byte>* host = nullptr; // a host buffer (blobs, __meta__)
};

// Streams one checkpoint file, header included, through a few pinned windows
// (memory stays bounded whatever the file size: C2's optimizer file is 84 GB).
// A reader thread preads window i+1 while window i goes to HBM in one DMA.
// There the GPU checksums it (lzk_fnv1a64_continue): every entry slice
// continues that entry's FNV-1a state, and optionally the whole window
// continues the whole-file digest (the manifest digest). Slices with a device
// sink are then scattered device-to-device; host sinks are copied from the
// pinned window. No byte is hashed on the host.
class FileStreamer {
 public:
  static constexpr uint64_t kWindow = 512ull << 20;
  static constexpr int kWindows = 3;

  explicit FileStreamer(int device);
  ~FileStreamer();
  FileStreamer(const FileStreamer&) = delete;
  FileStreamer& operator=(const FileStreamer&) = delete;

  // Streams bytes [0, header.payload_end()) of `path`. Returns the keys whose
  // checksum mismatches, in header order. `file_digest` (optional) receives
  // the FNV-1a-64 of those bytes.
  std::vector<std::string> run(const std::filesystem::path& path, const CheckpointFileHeader& header,
                               const std::vector<EntrySink>& sinks, uint64_t* file_digest = nullptr);
  // FNV-1a-64 and length of any whole file (no header needed).
  uint64_t digest(const std::filesystem::path& path, uint64_t* length);

  // Streamers are pooled per device: pinned and device windows stay
  // allocated between restores and commits (first-use allocation of the
  // windows costs hundreds of ms). The handle returns it to the pool.
  struct Release {
    void operator()(FileStreamer* s) const;
  };
  using Handle = std::unique_ptr<FileStreamer, Release>;
  static Handle acquire(int device);
  // Frees the idle pooled streamers (their pinned and device windows).
  static void trim();

 private:
  struct Window {
    std::byte* buf = nullptr;   // pinned host
    std::byte* dbuf = nullptr;  // device copy of the window
    uint64_t cap = 0;
    lzk_event* done = nullptr;
    bool used = false;
  };
  struct Range {
    uint64_t begin, end;  // file offsets
    const EntrySink* sink;
  };
  // Streams [0, end) of an open file: ranges are checksummed into
  // states_[0..ranges), the whole stream into states_[ranges] if `whole`.
  void stream(int fd, const std::filesystem::path& path, uint64_t end, const std::vector<Range>& ranges, bool whole);
  void ensure_states(size_t n);

  int device_;
  lzk_stream* stream_ = nullptr;
  Window win_[kWindows];
  uint64_t* states_ = nullptr;  // mapped host memory, written by the GPU
  size_t states_cap_ = 0;
};

}  // namespace lzckpt::detail
