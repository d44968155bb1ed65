// Uplink relay; see relay.hpp.
#include "relay.hpp"

#include <fcntl.h>
#include <sys/socket.h>
#include <sys/un.h>
#include <unistd.h>

#include <algorithm>
#include <cerrno>
#include <chrono>
#include <cstring>

#include "lzckpt/errors.hpp"

namespace lzckpt::detail {

namespace {

constexpr uint32_t kReq = 1, kReadDone = 2, kPersisted = 3;

void check(int rc, const char* what) {
  if (rc != LZK_OK) throw DeviceError(std::string(what) + ": " + lzk_last_error());
}

bool send_all(int fd, const void* p, size_t n) {
  const char* c = static_cast<const char*>(p);
  while (n) {
    const ssize_t w = ::send(fd, c, n, MSG_NOSIGNAL);
    if (w < 0 && errno == EINTR) continue;
    if (w <= 0) return false;
    c += w;
    n -= size_t(w);
  }
  return true;
}

bool recv_all(int fd, void* p, size_t n) {
  char* c = static_cast<char*>(p);
  while (n) {
    const ssize_t r = ::recv(fd, c, n, 0);
    if (r < 0 && errno == EINTR) continue;
    if (r <= 0) return false;
    c += r;
    n -= size_t(r);
  }
  return true;
}

// Frames: u32 type, u32 0, u64 payload length, payload.
struct Out {
  std::vector<std::byte> b;
  template <class T>
  void put(const T& v) {
    const auto* p = reinterpret_cast<const std::byte*>(&v);
    b.insert(b.end(), p, p + sizeof(T));
  }
  void bytes(const void* p, size_t n) {
    const auto* q = static_cast<const std::byte*>(p);
    b.insert(b.end(), q, q + n);
  }
};

struct In {
  const std::vector<std::byte>& b;
  size_t at = 0;
  template <class T>
  T get() {
    if (at + sizeof(T) > b.size()) throw Error("relay: truncated frame");
    T v;
    std::memcpy(&v, b.data() + at, sizeof(T));
    at += sizeof(T);
    return v;
  }
  std::string str(size_t n) {
    if (at + n > b.size()) throw Error("relay: truncated frame");
    std::string s(reinterpret_cast<const char*>(b.data() + at), n);
    at += n;
    return s;
  }
};

bool send_frame(int fd, uint32_t type, const std::vector<std::byte>& payload) {
  const uint32_t hdr[2] = {type, 0};
  const uint64_t len = payload.size();
  return send_all(fd, hdr, sizeof hdr) && send_all(fd, &len, sizeof len) &&
         (payload.empty() || send_all(fd, payload.data(), payload.size()));
}

bool recv_frame(int fd, uint32_t& type, std::vector<std::byte>& payload) {
  uint32_t hdr[2];
  uint64_t len = 0;
  if (!recv_all(fd, hdr, sizeof hdr) || !recv_all(fd, &len, sizeof len)) return false;
  if (len > (1ull << 30)) return false;
  type = hdr[0];
  payload.resize(len);
  return len == 0 || recv_all(fd, payload.data(), len);
}

sockaddr_un address(const std::string& path) {
  sockaddr_un a{};
  a.sun_family = AF_UNIX;
  if (path.size() >= sizeof a.sun_path) throw ConfigError("relay socket path too long: " + path);
  std::memcpy(a.sun_path, path.c_str(), path.size() + 1);
  return a;
}

void pwrite_all(int fd, const std::byte* p, uint64_t n, uint64_t off, const std::string& path) {
  while (n) {
    const ssize_t w = ::pwrite(fd, p, n, off_t(off));
    if (w < 0 && errno == EINTR) continue;
    if (w <= 0) throw IoError("relay: write to " + path + " failed: " + std::strerror(errno));
    p += w;
    n -= uint64_t(w);
    off += uint64_t(w);
  }
}

}  // namespace

// ---------------------------------------------------------------------------
// helper side

struct RelayServer::Request {
  uint64_t id = 0;
  uint32_t flags = 0;
  bool has_producer = false;
  lzk_ipc_handle producer{};
  std::string path;
  std::vector<RelayEntry> entries;
  std::chrono::steady_clock::time_point received{};
};

RelayServer::RelayServer(int device, std::string socket_path, uint64_t staging_bytes, uint32_t ctas,
                         bool copy_engines)
    : device_(device),
      path_(std::move(socket_path)),
      chunk_(std::clamp<uint64_t>(staging_bytes / 4, 1ull << 20, 256ull << 20) & ~uint64_t(4095)),
      ctas_(ctas ? ctas : 4),
      copy_engines_(copy_engines) {
  check(lzk_set_device(device_), "relay server: device");
  check(lzk_stream_create(device_, 0, &stream_), "relay server: stream");
  check(lzk_stream_create(device_, 0, &hash_stream_), "relay server: hash stream");
  if (copy_engines_) check(lzk_stream_create(device_, 0, &pull_stream_), "relay server: pull stream");
  const size_t slots = size_t(std::max<uint64_t>(2, staging_bytes / chunk_));
  for (size_t k = 0; k < slots; ++k) {
    void* p = nullptr;
    check(lzk_host_alloc(chunk_, LZK_HOST_MAPPED | LZK_HOST_HUGEPAGE, &p), "relay server: staging");
    staging_.push_back(static_cast<std::byte*>(p));
    lzk_event* e = nullptr;
    check(lzk_event_create(device_, 1, &e), "relay server: event");
    chunk_done_.push_back(e);
    if (copy_engines_) {
      void* d = nullptr;
      check(lzk_dev_alloc(device_, chunk_, &d), "relay server: HBM staging");
      dev_stage_.push_back(d);
      lzk_event* pe = nullptr;
      check(lzk_event_create(device_, 0, &pe), "relay server: event");
      pulled_.push_back(pe);
    }
  }
  listen_fd_ = ::socket(AF_UNIX, SOCK_STREAM | SOCK_CLOEXEC, 0);
  if (listen_fd_ < 0) throw IoError("relay server: socket() failed");
  const sockaddr_un a = address(path_);
  ::unlink(path_.c_str());
  if (::bind(listen_fd_, reinterpret_cast<const sockaddr*>(&a), sizeof a) != 0 || ::listen(listen_fd_, 16) != 0) {
    ::close(listen_fd_);
    throw IoError("relay server: cannot listen on " + path_ + ": " + std::strerror(errno));
  }
  acceptor_ = std::thread([this] { accept_loop(); });
}

RelayServer::~RelayServer() {
  {
    std::lock_guard lk(mu_);
    stop_ = true;
    for (int fd : conn_fds_) ::shutdown(fd, SHUT_RDWR);
  }
  ::shutdown(listen_fd_, SHUT_RDWR);
  ::close(listen_fd_);
  if (acceptor_.joinable()) acceptor_.join();
  for (auto& t : conns_) {
    if (t.joinable()) t.join();
  }
  for (int fd : conn_fds_) ::close(fd);
  ::unlink(path_.c_str());
  lzk_stream_sync(stream_);
  lzk_stream_sync(hash_stream_);
  if (pull_stream_) lzk_stream_sync(pull_stream_);
  for (auto* e : chunk_done_) lzk_event_destroy(e);
  for (auto* e : pulled_) lzk_event_destroy(e);
  for (void* d : dev_stage_) lzk_dev_free(device_, d);
  if (pull_stream_) lzk_stream_destroy(pull_stream_);
  for (auto& [k, e] : events_) lzk_event_destroy(e);
  for (auto* p : staging_) lzk_host_free(p);
  if (digests_) lzk_host_free(digests_);
  lzk_stream_destroy(hash_stream_);
  lzk_stream_destroy(stream_);
}

uint64_t RelayServer::bytes_relayed() const {
  std::lock_guard lk(mu_);
  return bytes_;
}

uint64_t RelayServer::requests() const {
  std::lock_guard lk(mu_);
  return requests_;
}

void RelayServer::accept_loop() {
  for (;;) {
    const int fd = ::accept4(listen_fd_, nullptr, nullptr, SOCK_CLOEXEC);
    if (fd < 0) {
      if (errno == EINTR) continue;
      return;  // shut down
    }
    std::lock_guard lk(mu_);
    if (stop_) {
      ::close(fd);
      return;
    }
    conn_fds_.push_back(fd);
    conns_.emplace_back([this, fd] { serve(fd); });
  }
}

void RelayServer::serve(int fd) {
  lzk_set_device(device_);
  std::vector<std::byte> payload;
  uint32_t type = 0;
  while (recv_frame(fd, type, payload)) {
    if (type != kReq) return;
    Request r;
    try {
      In in{payload};
      r.id = in.get<uint64_t>();
      r.flags = in.get<uint32_t>();
      const uint32_t n = in.get<uint32_t>();
      r.has_producer = in.get<uint32_t>() != 0;
      r.producer = in.get<lzk_ipc_handle>();
      const uint32_t plen = in.get<uint32_t>();
      r.path = in.str(plen);
      r.entries.resize(n);
      for (auto& e : r.entries) e = in.get<RelayEntry>();
    } catch (const std::exception&) {
      return;  // malformed: drop the connection
    }
    r.received = std::chrono::steady_clock::now();
    std::lock_guard lk(mu_);
    if (stop_) return;
    handle(fd, r);
  }
}

// One request, under mu_: producer wait, optional device FNV of the sources,
// gather through the staging ring (each chunk written out while later ones
// are gathered), READ_DONE once every read of the owner's memory is done,
// then the remaining writes, fsync and PERSISTED.
void RelayServer::handle(int fd, Request& r) {
  const auto started = std::chrono::steady_clock::now();
  bool read_sent = false;
  auto reply = [&](uint32_t type, bool ok, const std::string& err, const std::vector<uint64_t>& sums) {
    Out o;
    o.put(r.id);
    o.put(uint32_t(ok));
    if (type == kPersisted) {
      o.put(uint32_t(sums.size()));
      for (uint64_t v : sums) o.put(v);
    }
    o.put(uint32_t(err.size()));
    o.bytes(err.data(), err.size());
    send_frame(fd, type, o.b);
  };
  int file = -1;
  try {
    const size_t n = r.entries.size();
    // Mappings of the owners' allocations are kept between requests; an
    // owner that frees and re-allocates tensors produces new handles, and the
    // old mappings would pin its freed memory. Drop them all past a bound
    // (no request is in flight here: requests are handled one at a time).
    for (const auto& e : r.entries) {
      opened_.insert(std::string(reinterpret_cast<const char*>(&e.mem), sizeof e.mem));
    }
    if (opened_.size() > kMaxOpen) {
      lzk_ipc_close_all();
      opened_.clear();
      for (const auto& e : r.entries) {
        opened_.insert(std::string(reinterpret_cast<const char*>(&e.mem), sizeof e.mem));
      }
    }
    std::vector<const std::byte*> src(n);
    for (size_t i = 0; i < n; ++i) {
      void* base = nullptr;
      check(lzk_ipc_open_mem(device_, &r.entries[i].mem, &base), "relay: open the owner's allocation");
      src[i] = static_cast<const std::byte*>(base) + r.entries[i].src_offset;
    }
    if (r.has_producer) {
      const std::string key(reinterpret_cast<const char*>(&r.producer), sizeof r.producer);
      auto it = events_.find(key);
      if (it == events_.end()) {
        lzk_event* e = nullptr;
        check(lzk_ipc_event_open(device_, &r.producer, &e), "relay: open the producer event");
        it = events_.emplace(key, e).first;
      }
      check(lzk_stream_wait_event(stream_, it->second), "relay: producer wait");
      if (pull_stream_) check(lzk_stream_wait_event(pull_stream_, it->second), "relay: producer wait");
      if (r.flags & kRelayHash) check(lzk_stream_wait_event(hash_stream_, it->second), "relay: producer wait");
    }
    std::vector<uint64_t> sums;
    if (r.flags & kRelayHash) {
      if (digest_cap_ < n) {
        if (digests_) lzk_host_free(digests_);
        void* p = nullptr;
        check(lzk_host_alloc(std::max<size_t>(n, 64) * 8, LZK_HOST_MAPPED, &p), "relay: digests");
        digests_ = static_cast<uint64_t*>(p);
        digest_cap_ = uint32_t(std::max<size_t>(n, 64));
      }
      std::vector<lzk_hash_desc> hd(n);
      for (size_t i = 0; i < n; ++i) {
        hd[i] = {reinterpret_cast<uint64_t>(src[i]), r.entries[i].length, LZK_FNV_BASIS,
                 reinterpret_cast<uint64_t>(digests_ + i)};
      }
      // on its own stream, concurrently with the gathers below
      check(lzk_fnv1a64_batch(hash_stream_, hd.data(), uint32_t(n), 16), "relay: entry checksums");
    }
    if (r.flags & kRelayWrite) {
      file = ::open(r.path.c_str(), O_WRONLY | O_CLOEXEC);
      if (file < 0) throw IoError("relay: cannot open " + r.path + ": " + std::strerror(errno));
    }
    // the byte stream of all entries, cut into staging chunks
    struct Piece {
      uint64_t file_off, len, stage_off;
    };
    const size_t slots = staging_.size();
    std::vector<std::vector<Piece>> slot_pieces(slots);
    std::vector<bool> slot_busy(slots, false);
    auto retire = [&](size_t k) {
      if (!slot_busy[k]) return;
      check(lzk_event_sync(chunk_done_[k]), "relay: gather");
      if (file >= 0) {
        for (const auto& p : slot_pieces[k]) pwrite_all(file, staging_[k] + p.stage_off, p.len, p.file_off, r.path);
      }
      slot_pieces[k].clear();
      slot_busy[k] = false;
    };
    size_t ei = 0, slot = 0;
    uint64_t eoff = 0, total = 0;
    while (ei < n) {
      retire(slot);
      std::vector<lzk_copy_desc> descs;
      uint64_t used = 0;
      while (ei < n && used < chunk_) {
        const RelayEntry& e = r.entries[ei];
        const uint64_t take = std::min(e.length - eoff, chunk_ - used);
        if (take) {
          descs.push_back({reinterpret_cast<uint64_t>(src[ei] + eoff), reinterpret_cast<uint64_t>(staging_[slot] + used),
                           take});
          slot_pieces[slot].push_back({e.file_offset + eoff, take, used});
        }
        used += take;
        eoff += take;
        if (eoff == e.length) {
          ++ei;
          eoff = 0;
        }
      }
      if (!descs.empty()) {
        if (copy_engines_) {
          // pull over NVLink into HBM (D2D), then one DMA over this GPU's link;
          // slot reuse is safe: retire(slot) above waited for its last DMA
          auto* dst = static_cast<std::byte*>(dev_stage_[slot]);
          for (auto& d : descs) d.dst = reinterpret_cast<uint64_t>(dst) + (d.dst - reinterpret_cast<uint64_t>(staging_[slot]));
          check(lzk_ce_copy_d2d(pull_stream_, descs.data(), uint32_t(descs.size())), "relay: pull");
          check(lzk_event_record(pulled_[slot], pull_stream_), "relay: event");
          check(lzk_stream_wait_event(stream_, pulled_[slot]), "relay: pull wait");
          const lzk_copy_desc out{reinterpret_cast<uint64_t>(dst), reinterpret_cast<uint64_t>(staging_[slot]), used};
          check(lzk_ce_copy_d2h(stream_, &out, 1), "relay: push");
        } else {
          check(lzk_gather_d2h(stream_, descs.data(), uint32_t(descs.size()), ctas_), "relay: gather");
        }
        check(lzk_event_record(chunk_done_[slot], stream_), "relay: event");
        slot_busy[slot] = true;
        total += used;
      }
      slot = (slot + 1) % slots;
    }
    check(lzk_stream_sync(stream_), "relay: reads");  // every read of the owner's memory is done
    check(lzk_stream_sync(hash_stream_), "relay: checksums");
    if (trace_) {
      using ms = std::chrono::duration<double, std::milli>;
      const auto now = std::chrono::steady_clock::now();
      std::fprintf(stderr, "[relay] dev %d req %llu: %.1f MB in %zu entries, queued %.2f ms, read %.2f ms (%.1f GB/s), idle before %.2f ms\n",
                   device_, (unsigned long long)r.id, total / 1e6, n, ms(started - r.received).count(),
                   ms(now - started).count(), total / 1e6 / std::max(1e-9, ms(now - started).count()),
                   ms(started - last_done_).count());
      last_done_ = now;
    }
    if (r.flags & kRelayHash) sums.assign(digests_, digests_ + n);
    reply(kReadDone, true, "", {});
    read_sent = true;
    for (size_t k = 0; k < slots; ++k) retire((slot + k) % slots);  // remaining writes, oldest first
    if (file >= 0 && (r.flags & kRelayFsync) && ::fsync(file) != 0) {
      throw IoError("relay: fsync of " + r.path + " failed");
    }
    if (file >= 0) ::close(file);
    file = -1;
    bytes_ += total;
    ++requests_;
    if (!(r.flags & kRelayHash)) sums.assign(n, 0);
    reply(kPersisted, true, "", sums);
  } catch (const std::exception& e) {
    if (file >= 0) ::close(file);
    lzk_stream_sync(stream_);
    lzk_stream_sync(hash_stream_);
    if (!read_sent) reply(kReadDone, false, e.what(), {});
    reply(kPersisted, false, e.what(), {});
  }
}

// ---------------------------------------------------------------------------
// owner side

RelayClient::RelayClient(const std::string& socket_path) {
  const sockaddr_un a = address(socket_path);
  // the helper may still be starting: retry for a while
  for (int attempt = 0; attempt < 1200; ++attempt) {  // 120 s
    fd_ = ::socket(AF_UNIX, SOCK_STREAM | SOCK_CLOEXEC, 0);
    if (fd_ < 0) throw IoError("relay client: socket() failed");
    if (::connect(fd_, reinterpret_cast<const sockaddr*>(&a), sizeof a) == 0) break;
    ::close(fd_);
    fd_ = -1;
    std::this_thread::sleep_for(std::chrono::milliseconds(100));
  }
  if (fd_ < 0) throw IoError("relay client: no relay server at " + socket_path);
  reader_ = std::thread([this] { reader_loop(); });
}

RelayClient::~RelayClient() {
  ::shutdown(fd_, SHUT_RDWR);
  if (reader_.joinable()) reader_.join();
  ::close(fd_);
}

bool RelayClient::connected() const {
  std::lock_guard lk(mu_);
  return !broken_;
}

void RelayClient::submit(const std::filesystem::path& file, uint32_t flags, const lzk_ipc_handle* producer,
                         const std::vector<RelayEntry>& entries, ReadDone on_read, Persisted on_persisted) {
  uint64_t id;
  {
    std::lock_guard lk(mu_);
    if (broken_) throw IoError("relay: connection to the helper is lost");
    id = next_++;
    pending_[id] = Pending{std::move(on_read), std::move(on_persisted), false, std::chrono::steady_clock::now()};
  }
  Out o;
  o.put(id);
  o.put(flags);
  o.put(uint32_t(entries.size()));
  o.put(uint32_t(producer != nullptr));
  lzk_ipc_handle none{};
  o.put(producer ? *producer : none);
  const std::string p = file.string();
  o.put(uint32_t(p.size()));
  o.bytes(p.data(), p.size());
  for (const auto& e : entries) o.put(e);
  bool sent;
  {
    std::lock_guard lk(send_mu_);
    sent = send_frame(fd_, kReq, o.b);
  }
  if (!sent) {
    std::lock_guard lk(mu_);
    pending_.erase(id);
    throw IoError("relay: cannot reach the helper");
  }
}

void RelayClient::fail_all(const std::string& why) {
  std::map<uint64_t, Pending> dead;
  {
    std::lock_guard lk(mu_);
    broken_ = true;
    dead.swap(pending_);
  }
  for (auto& [id, p] : dead) {
    if (!p.read && p.on_read) p.on_read(false, why);
    if (p.on_persisted) p.on_persisted(false, why, {});
  }
}

void RelayClient::reader_loop() {
  std::vector<std::byte> payload;
  uint32_t type = 0;
  while (recv_frame(fd_, type, payload)) {
    try {
      In in{payload};
      const uint64_t id = in.get<uint64_t>();
      const bool ok = in.get<uint32_t>() != 0;
      std::vector<uint64_t> sums;
      if (type == kPersisted) {
        const uint32_t n = in.get<uint32_t>();
        sums.resize(n);
        for (auto& v : sums) v = in.get<uint64_t>();
      }
      const std::string err = in.str(in.get<uint32_t>());
      Pending p;
      {
        std::lock_guard lk(mu_);
        auto it = pending_.find(id);
        if (it == pending_.end()) continue;
        if (type == kReadDone) {
          it->second.read = true;
          p.on_read = it->second.on_read;
          if (trace_) {
            std::fprintf(stderr, "[relay-owner] req %llu: READ_DONE %.2f ms after submit\n", (unsigned long long)id,
                         std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - it->second.sent)
                             .count());
          }
        } else {
          p = std::move(it->second);
          pending_.erase(it);
        }
      }
      if (type == kReadDone && p.on_read) p.on_read(ok, err);
      if (type == kPersisted && p.on_persisted) p.on_persisted(ok, err, sums);
    } catch (const std::exception&) {
      break;
    }
  }
  fail_all("relay: connection to the helper closed");
}

}  // namespace lzckpt::detail
