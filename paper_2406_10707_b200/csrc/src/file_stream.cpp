// See file_stream.hpp.
#include "file_stream.hpp"

#include <fcntl.h>
#include <sys/mman.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cerrno>
#include <cstring>
#include <exception>
#include <mutex>
#include <thread>

#include "lzckpt/checksum.hpp"
#include "lzckpt/errors.hpp"

namespace lzckpt::detail {

void ck(int rc, const char* what) {
  if (rc != LZK_OK) throw DeviceError(std::string(what) + ": " + lzk_last_error());
}

namespace {

// Window reads from the disk (O_DIRECT): 2 concurrent preads of 16 MiB. On
// the GPU boxes' virtio disk that reads 6.0 GB/s against 4.0 for 8 x 64 MiB
// (profiles/r02_disk_read_probe.txt) and restores a C2 sample at 3.55 GB/s
// median against 3.25 (r02_restore_probe.txt). Windows already in the page
// cache are memcpys: 8 threads x 64 MiB. LZCKPT_READ_THREADS /
// LZCKPT_READ_PIECE_MB override the disk setting (tools/restore_read_probe.py).
unsigned env_uint(const char* name, unsigned dflt) {
  const char* v = std::getenv(name);
  return v && std::atoi(v) > 0 ? unsigned(std::atoi(v)) : dflt;
}
unsigned read_threads(bool direct) {
  static const unsigned n = env_uint("LZCKPT_READ_THREADS", 2);
  return direct ? n : 8;
}
uint64_t read_piece(bool direct) {
  static const uint64_t n = uint64_t(env_uint("LZCKPT_READ_PIECE_MB", 16)) << 20;
  return direct ? n : 64ull << 20;
}

// Runs fn(i) for i in [0, n) on up to `threads` threads.
template <class Fn>
void parallel_for(size_t n, unsigned threads, Fn fn) {
  if (n == 0) return;
  threads = unsigned(std::min<size_t>(threads, n));
  if (threads <= 1) {
    for (size_t i = 0; i < n; ++i) fn(i);
    return;
  }
  std::atomic<size_t> next{0};
  std::vector<std::thread> th;
  std::exception_ptr err;
  std::mutex err_mu;
  for (unsigned t = 0; t < threads; ++t) {
    th.emplace_back([&] {
      for (size_t i; (i = next.fetch_add(1)) < n;) {
        try {
          fn(i);
        } catch (...) {
          std::lock_guard lk(err_mu);
          if (!err) err = std::current_exception();
        }
      }
    });
  }
  for (auto& t : th) t.join();
  if (err) std::rethrow_exception(err);
}

void pread_all(int fd, void* dst, uint64_t n, uint64_t off, const std::filesystem::path& p) {
  auto* d = static_cast<char*>(dst);
  while (n) {
    ssize_t r = ::pread(fd, d, n, off_t(off));
    if (r < 0 && errno == EINTR) continue;
    if (r <= 0) throw IoError("read failed for " + p.string());
    d += r;
    off += uint64_t(r);
    n -= uint64_t(r);
  }
}

// O_DIRECT read of [off, off + n) into an aligned buffer (off aligned to
// 4 KiB; n rounded up to a block, a short read at EOF is fine). Returns
// false when the file system refuses O_DIRECT (caller reads buffered).
bool pread_direct(int dfd, void* dst, uint64_t n, uint64_t off, uint64_t file_end) {
  constexpr uint64_t kBlock = 4096;
  if (dfd < 0 || off % kBlock || reinterpret_cast<uintptr_t>(dst) % kBlock) return false;
  const uint64_t want = (n + kBlock - 1) & ~(kBlock - 1);
  auto* d = static_cast<char*>(dst);
  uint64_t done = 0;
  while (done < n) {
    const ssize_t r = ::pread(dfd, d + done, want - done, off_t(off + done));
    if (r < 0) {
      if (errno == EINTR) continue;
      if (errno == EINVAL && done == 0) return false;
      throw IoError("read failed: " + std::string(std::strerror(errno)));
    }
    if (r == 0) break;
    done += uint64_t(r);
  }
  if (done < n && off + done < file_end) throw IoError("short O_DIRECT read");
  return true;
}

struct Fd {
  int fd;
  ~Fd() {
    if (fd >= 0) ::close(fd);
  }
};

}  // namespace

FileStreamer::FileStreamer(int device) : device_(device) {
  ck(lzk_stream_create(device, 0, &stream_), "file stream");
  for (auto& w : win_) ck(lzk_event_create(device, 1, &w.done), "file stream event");
}

FileStreamer::~FileStreamer() {
  for (auto& w : win_) {
    if (w.done) lzk_event_destroy(w.done);
    lzk_host_free(w.buf);
    lzk_dev_free(device_, w.dbuf);
  }
  lzk_host_free(states_);
  lzk_stream_destroy(stream_);
}

namespace {
std::mutex g_pool_mu;
std::vector<FileStreamer*> g_pool;  // idle streamers (any device)
constexpr size_t kPoolMax = 4;
}  // namespace

FileStreamer::Handle FileStreamer::acquire(int device) {
  {
    std::lock_guard lk(g_pool_mu);
    for (size_t i = 0; i < g_pool.size(); ++i) {
      if (g_pool[i]->device_ == device) {
        FileStreamer* s = g_pool[i];
        g_pool.erase(g_pool.begin() + long(i));
        return Handle(s);
      }
    }
  }
  return Handle(new FileStreamer(device));
}

void FileStreamer::Release::operator()(FileStreamer* s) const {
  std::lock_guard lk(g_pool_mu);
  if (g_pool.size() < kPoolMax) {
    g_pool.push_back(s);
    return;
  }
  delete s;
}

void FileStreamer::trim() {
  std::vector<FileStreamer*> idle;
  {
    std::lock_guard lk(g_pool_mu);
    idle.swap(g_pool);
  }
  for (auto* s : idle) delete s;
}

void FileStreamer::ensure_states(size_t n) {
  if (states_cap_ >= n) return;
  lzk_host_free(states_);
  states_ = nullptr;
  void* p = nullptr;
  ck(lzk_host_alloc(std::max<size_t>(n, 1) * 8, LZK_HOST_MAPPED, &p), "file stream digests");
  states_ = static_cast<uint64_t*>(p);
  states_cap_ = n;
}

void FileStreamer::stream(int fd, const std::filesystem::path& path, uint64_t end, const std::vector<Range>& ranges,
                          bool whole) {
  Fd direct{::open(path.c_str(), O_RDONLY | O_DIRECT | O_CLOEXEC)};  // -1: buffered reads only
  const int dfd = direct.fd;
  // Page-cache residency per window (mincore on a read-only mapping): a
  // window mostly in the cache is read through it, anything else with
  // O_DIRECT (durable writes bypass the cache, so fresh checkpoints are cold).
  void* map = end ? ::mmap(nullptr, end, PROT_READ, MAP_SHARED, fd, 0) : MAP_FAILED;
  struct Unmap {
    void* p;
    uint64_t n;
    ~Unmap() {
      if (p != MAP_FAILED) ::munmap(p, n);
    }
  } unmap{map, end};
  auto mostly_cached = [&](uint64_t off, uint64_t len) {
    if (map == MAP_FAILED || len == 0) return true;
    const uint64_t pg = 4096, npg = (len + pg - 1) / pg;
    std::vector<unsigned char> v(npg);
    if (::mincore(static_cast<char*>(map) + off, len, v.data()) != 0) return true;
    uint64_t res = 0;
    for (unsigned char c : v) res += c & 1;
    return res * 2 >= npg;
  };
  NvtxRange range("lzckpt.file_stream");
  PhaseTrace tr("file_stream");
  // a previous call that failed midway may have left DMAs in flight
  ck(lzk_stream_sync(stream_), "file stream drain");
  const uint64_t wsize = std::min(kWindow, std::max<uint64_t>(end, 1));
  const size_t slots = size_t(std::min<uint64_t>(kWindows, (end + wsize - 1) / wsize));
  for (size_t k = 0; k < size_t(kWindows); ++k) {
    Window& w = win_[k];
    if (k < slots && w.cap < wsize) {
      lzk_host_free(w.buf);
      w.buf = nullptr;
      lzk_dev_free(device_, w.dbuf);
      w.dbuf = nullptr;
      void* p = nullptr;
      ck(lzk_host_alloc(wsize, LZK_HOST_MAPPED | LZK_HOST_HUGEPAGE, &p), "file stream window");
      w.buf = static_cast<std::byte*>(p);
      ck(lzk_dev_alloc(device_, wsize, &p), "file stream device window");
      w.dbuf = static_cast<std::byte*>(p);
      w.cap = wsize;
    }
    w.used = false;
  }
  const size_t nr = ranges.size();
  ensure_states(nr + 1);
  for (size_t e = 0; e <= nr; ++e) states_[e] = Fnv64::kOffset;
  tr.mark("setup");
  double wait_read = 0, t_h2d = 0, t_hash = 0, t_d2d = 0;
  const size_t nwin = size_t((end + wsize - 1) / wsize);
  // reader: window i -> slot i % kWindows (waits until the slot's DMA finished)
  auto read_window = [&](size_t i) {
    Window& w = win_[i % kWindows];
    if (w.used) ck(lzk_event_sync(w.done), "file stream window reuse");
    const uint64_t off = uint64_t(i) * wsize, len = std::min(wsize, end - off);
    const bool use_direct = dfd >= 0 && !mostly_cached(off, len);
    const uint64_t piece = read_piece(use_direct);
    parallel_for(size_t((len + piece - 1) / piece), read_threads(use_direct), [&](size_t k) {
      const uint64_t o = uint64_t(k) * piece, n = std::min(piece, len - o);
      // O_DIRECT first (files written by the flush are usually not in the
      // page cache); windows are page-aligned and piece offsets multiples of
      // the (MiB-sized) piece. The round-up of the last piece stays inside the window.
      if (!(use_direct && o + ((n + 4095) & ~uint64_t(4095)) <= w.cap && pread_direct(dfd, w.buf + o, n, off + o, end))) {
        pread_all(fd, w.buf + o, n, off + o, path);
      }
    });
  };
  std::thread reader;
  std::exception_ptr read_err;
  struct JoinOnUnwind {  // an exception below must not destroy a joinable reader
    std::thread& t;
    ~JoinOnUnwind() {
      if (t.joinable()) t.join();
    }
  } join_guard{reader};
  if (nwin) read_window(0);
  tr.mark("read0");
  for (size_t i = 0; i < nwin; ++i) {
    const auto tw = std::chrono::steady_clock::now();
    if (reader.joinable()) reader.join();
    wait_read += since(tw);
    if (read_err) std::rethrow_exception(read_err);
    Window& w = win_[i % kWindows];
    const uint64_t off = uint64_t(i) * wsize, len = std::min(wsize, end - off);
    lzk_copy_desc up{reinterpret_cast<uint64_t>(w.buf), reinterpret_cast<uint64_t>(w.dbuf), len};
    ck(lzk_ce_copy_h2d(stream_, &up, 1), "file stream DMA");
    ck(lzk_event_record(w.done, stream_), "file stream event");  // host window reusable after this
    w.used = true;
    if (i + 1 < nwin) {
      reader = std::thread([&, i] {
        try {
          read_window(i + 1);
        } catch (...) {
          read_err = std::current_exception();
        }
      });
    }
    std::vector<lzk_hash_desc> hd;
    std::vector<lzk_copy_desc> d2d;
    if (whole) hd.push_back({reinterpret_cast<uint64_t>(w.dbuf), len, 0, reinterpret_cast<uint64_t>(states_ + nr)});
    for (size_t e = 0; e < nr; ++e) {
      const Range& r = ranges[e];
      const uint64_t a = std::max(r.begin, off), b = std::min(r.end, off + len);
      if (a >= b) continue;
      const uint64_t src = reinterpret_cast<uint64_t>(w.dbuf + (a - off));
      hd.push_back({src, b - a, 0, reinterpret_cast<uint64_t>(states_ + e)});
      if (!r.sink) continue;
      if (r.sink->device) {
        d2d.push_back({src, reinterpret_cast<uint64_t>(static_cast<std::byte*>(r.sink->device) + (a - r.begin)), b - a});
      } else if (r.sink->host) {
        std::memcpy(r.sink->host->data() + (a - r.begin), w.buf + (a - off), b - a);
      }
    }
    auto gpu_mark = [&](double& acc) {  // trace only: serializes the pipeline
      if (!tr.on) return;
      const auto t0 = std::chrono::steady_clock::now();
      ck(lzk_stream_sync(stream_), "file stream trace sync");
      acc += since(t0);
    };
    gpu_mark(t_h2d);
    if (!hd.empty()) ck(lzk_fnv1a64_continue(stream_, hd.data(), uint32_t(hd.size()), 0), "file stream checksums");
    gpu_mark(t_hash);
    if (!d2d.empty()) ck(lzk_gather_d2d(stream_, d2d.data(), uint32_t(d2d.size()), 0), "file stream scatter");
    gpu_mark(t_d2d);
  }
  if (reader.joinable()) reader.join();
  if (read_err) std::rethrow_exception(read_err);
  tr.mark("windows");
  ck(lzk_stream_sync(stream_), "file stream sync");
  tr.mark("sync");
  if (tr.on) {
    tr.line += " read_wait=" + std::to_string(wait_read * 1e3) + " h2d=" + std::to_string(t_h2d * 1e3) +
               " hash=" + std::to_string(t_hash * 1e3) + " d2d=" + std::to_string(t_d2d * 1e3) +
               " nwin=" + std::to_string(nwin);
  }
}

std::vector<std::string> FileStreamer::run(const std::filesystem::path& path, const CheckpointFileHeader& h,
                                           const std::vector<EntrySink>& sinks, uint64_t* file_digest) {
  Fd f{::open(path.c_str(), O_RDONLY | O_CLOEXEC)};
  if (f.fd < 0) throw IoError("cannot open " + path.string());
  std::vector<Range> ranges(h.entries.size());
  for (size_t e = 0; e < h.entries.size(); ++e) {
    ranges[e] = {h.entries[e].offset, h.entries[e].offset + h.entries[e].length,
                 e < sinks.size() ? &sinks[e] : nullptr};
  }
  stream(f.fd, path, h.payload_end(), ranges, file_digest != nullptr);
  std::vector<std::string> bad;
  for (size_t e = 0; e < h.entries.size(); ++e) {
    if (states_[e] != h.entries[e].checksum) bad.push_back(h.entries[e].key);
  }
  if (file_digest) *file_digest = states_[h.entries.size()];
  return bad;
}

uint64_t FileStreamer::digest(const std::filesystem::path& path, uint64_t* length) {
  Fd f{::open(path.c_str(), O_RDONLY | O_CLOEXEC)};
  if (f.fd < 0) throw IoError("cannot open " + path.string());
  const off_t size = ::lseek(f.fd, 0, SEEK_END);
  if (size < 0) throw IoError("cannot stat " + path.string());
  stream(f.fd, path, uint64_t(size), {}, true);
  *length = uint64_t(size);
  return states_[0];
}

}  // namespace lzckpt::detail
