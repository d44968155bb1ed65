// B200 (sm_100a) device layer behind include/lzk_cuda.h.
//
// The hot kernel is lzk_gather_kernel: a multi-tensor gather copy that moves
// many device tensors into byte-granular offsets of a pinned, mapped host
// ring in ONE launch. It replaces the reference's per-chunk memcpy loop
// (reference proj/core/src/transfer_engine.cpp:117-160) and the per-leaf
// clone_bytes of small leaves at capture (proj/core/src/engine.cpp:138-143).
//
// Design:
//  * Descriptors travel as a __grid_constant__ kernel parameter (<= 32 KB),
//    so the call needs no staging buffer and the caller's array is free the
//    moment the launch returns. Larger batches become several launches.
//  * Work unit = a warp tile: <= kTile (16 KB) bytes of one descriptor owned
//    by one warp (16 per CTA), so many small tensors are copied in parallel
//    by a small grid. Tile boundaries sit at 128-byte-aligned DESTINATION
//    addresses: only a descriptor's first tile has an unaligned head and only
//    its last a tail.
//  * Loads: aligned 128-bit LDG of the source; when source and destination
//    disagree mod 16, each output word is funnel-shifted out of two adjacent
//    aligned source words (the neighbour's word hits L1).
//  * Stores: aligned 128-bit STG; a warp writes 512 contiguous bytes that
//    start on a 128-byte line = four full-line posted PCIe writes (ncu showed
//    16-byte-aligned warp stores straddling five lines cost ~15% of the link).
//  * Grid: a handful of CTAs saturates PCIe Gen5 x16 (measured: 2 CTAs for
//    >= 1 MiB tensors; warp tiles keep 4-KiB tensors link-bound with a small
//    grid too), so the snapshot steals only a few of the 148 SMs from
//    training kernels.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cctype>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include <sched.h>
#include <sys/mman.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <fstream>
#include <sstream>

#include <nvtx3/nvToolsExt.h>

#include "lzk_internal.h"

namespace lzk_detail {

thread_local std::string g_err;
std::atomic<uint64_t> launches{0};

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  cudaGetLastError();  // clear sticky-free errors so later calls are not poisoned
  if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) {
    return fail(LZK_ERR_NODEV, std::string(what) + ": " + cudaGetErrorString(e));
  }
  if (e == cudaErrorMemoryAllocation) {
    return fail(LZK_ERR_NOMEM, std::string(what) + ": " + cudaGetErrorString(e));
  }
  return fail(LZK_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

int use_device(int device) {
  int cur = -1;
  LZK_CK(cudaGetDevice(&cur));
  if (cur != device) LZK_CK(cudaSetDevice(device));
  return LZK_OK;
}

}  // namespace lzk_detail

namespace {

using lzk_detail::cuda_fail;
using lzk_detail::fail;
using lzk_detail::use_device;

// Per-thread, per-device non-blocking stream for the synchronous helpers.
cudaStream_t helper_stream(int device) {
  thread_local std::unordered_map<int, cudaStream_t> streams;
  auto it = streams.find(device);
  if (it != streams.end()) return it->second;
  cudaStream_t s = nullptr;
  if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) return nullptr;
  streams.emplace(device, s);
  return s;
}

// ---------------------------------------------------------------------------
// gather kernel
// ---------------------------------------------------------------------------

constexpr uint32_t kTile = 16u << 10;      // bytes of one descriptor per WARP work unit
constexpr int kThreads = 512;              // 16 warps per CTA
constexpr int kWarps = kThreads / 32;
constexpr int kUnroll = 4;                 // 16-byte words in flight per lane per pass
// Skewed copies hold two source words per output word: half the unroll keeps
// the kernel inside 128 registers (no spills) with ~256 KB still in flight
// across 8 CTAs, above the host link's bandwidth-delay product (~100 KB).
constexpr int kUnrollSkew = 2;
constexpr uint32_t kMaxDescPerLaunch = 960;

struct Desc {
  uint64_t src;
  uint64_t dst;
  uint64_t len;
  uint64_t tile_begin;  // exclusive prefix of tile counts
};

struct DescBatch {
  uint32_t n;
  uint32_t pad;
  uint64_t total_tiles;
  Desc d[kMaxDescPerLaunch];
};
static_assert(sizeof(DescBatch) <= 31 * 1024, "kernel parameter budget");

__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ uint4 ld_cached(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ void st_word(uint4* p, const uint4& v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

// out = bytes [4Q + r, 4Q + r + 16) of the 32-byte window (a, b); shift = 8r.
template <int Q>
__device__ __forceinline__ uint4 extract(const uint4& a, const uint4& b, uint32_t shift) {
  const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
  uint4 o;
  o.x = __funnelshift_r(w[Q + 0], w[Q + 1], shift);
  o.y = __funnelshift_r(w[Q + 1], w[Q + 2], shift);
  o.z = __funnelshift_r(w[Q + 2], w[Q + 3], shift);
  o.w = __funnelshift_r(w[Q + 3], w[Q + 4], shift);
  return o;
}

// Aligned-destination body, one warp: nw 16-byte words to dw from aligned
// source words sa at byte skew k in [1, 15]. Lane l owns words l, l+32, ...
template <int Q>
__device__ __forceinline__ void body_skewed(const uint4* __restrict__ sa, uint4* dw, uint32_t nw,
                                            uint32_t shift, uint32_t lane) {
  for (uint32_t base = lane; base < nw; base += 32 * kUnrollSkew) {
    uint4 lo[kUnrollSkew], hi[kUnrollSkew];
#pragma unroll
    for (int u = 0; u < kUnrollSkew; ++u) {
      const uint32_t j = base + u * 32;
      if (j < nw) {
        lo[u] = ld_cached(sa + j);
        hi[u] = ld_cached(sa + j + 1);
      }
    }
#pragma unroll
    for (int u = 0; u < kUnrollSkew; ++u) {
      const uint32_t j = base + u * 32;
      if (j < nw) st_word(dw + j, extract<Q>(lo[u], hi[u], shift));
    }
  }
}

__device__ __forceinline__ void body_aligned(const uint4* __restrict__ sw, uint4* dw, uint32_t nw, uint32_t lane) {
  for (uint32_t base = lane; base < nw; base += 32 * kUnroll) {
    uint4 v[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const uint32_t j = base + u * 32;
      if (j < nw) v[u] = ld_stream(sw + j);
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const uint32_t j = base + u * 32;
      if (j < nw) st_word(dw + j, v[u]);
    }
  }
}

__device__ __forceinline__ void copy_words(const uint8_t* s, uint4* dw, uint32_t nw, uint32_t lane) {
  const uint32_t k = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(s) & 15u);
  if (k == 0) {
    body_aligned(reinterpret_cast<const uint4*>(s), dw, nw, lane);
    return;
  }
  const uint4* sa = reinterpret_cast<const uint4*>(s - k);
  const uint32_t shift = 8u * (k & 3u);
  switch (k >> 2) {
    case 0: body_skewed<0>(sa, dw, nw, shift, lane); break;
    case 1: body_skewed<1>(sa, dw, nw, shift, lane); break;
    case 2: body_skewed<2>(sa, dw, nw, shift, lane); break;
    default: body_skewed<3>(sa, dw, nw, shift, lane); break;
  }
}

// One warp copies n bytes src -> dst. Stores are shaped for the host link:
// bytes up to the first 16-byte boundary go bytewise, then up to seven
// 16-byte words up to the first 128-byte line boundary, then the body, where
// every warp store covers 512 bytes starting on a line boundary (four
// full-line posted writes, never five partial ones), then the tail.
__device__ __forceinline__ void copy_span(const uint8_t* src, uint8_t* dst, uint64_t n, uint32_t lane) {
  uint32_t head = static_cast<uint32_t>((16u - (reinterpret_cast<uintptr_t>(dst) & 15u)) & 15u);
  if (head > n) head = static_cast<uint32_t>(n);
  if (lane < head) dst[lane] = src[lane];
  const uint8_t* s = src + head;
  uint8_t* d = dst + head;
  uint64_t rem = n - head;
  uint32_t lead = static_cast<uint32_t>(((128u - (reinterpret_cast<uintptr_t>(d) & 127u)) & 127u) >> 4);
  if (lead > (rem >> 4)) lead = static_cast<uint32_t>(rem >> 4);
  if (lead) {
    if (lane < lead) {
      const uint8_t* sw = s + 16u * lane;
      uint4 v;
      if ((reinterpret_cast<uintptr_t>(sw) & 15u) == 0) {
        v = ld_cached(reinterpret_cast<const uint4*>(sw));
      } else {
        uint32_t b[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          b[q] = uint32_t(sw[4 * q]) | (uint32_t(sw[4 * q + 1]) << 8) | (uint32_t(sw[4 * q + 2]) << 16) |
                 (uint32_t(sw[4 * q + 3]) << 24);
        }
        v = make_uint4(b[0], b[1], b[2], b[3]);
      }
      st_word(reinterpret_cast<uint4*>(d) + lane, v);
    }
    s += 16u * lead;
    d += 16u * lead;
    rem -= 16u * lead;
  }
  const uint32_t nw = static_cast<uint32_t>(rem >> 4);
  const uint32_t tail = static_cast<uint32_t>(rem & 15u);
  if (nw) copy_words(s, reinterpret_cast<uint4*>(d), nw, lane);
  if (lane < tail) {
    const uint64_t o = static_cast<uint64_t>(nw) * 16u + lane;
    d[o] = s[o];
  }
}

// Grid-stride over warp tiles: tile t of descriptor i covers destination
// bytes [local*kTile - mis, (local+1)*kTile - mis) clipped to the
// descriptor, mis = dst & 127, so interior boundaries sit on 128-byte lines.
// Each warp finds its descriptor by a warp-uniform binary search over the
// tile prefix (broadcast constant-bank reads).
__global__ void __launch_bounds__(kThreads)
    lzk_gather_kernel(const __grid_constant__ DescBatch batch) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint64_t warp = uint64_t(blockIdx.x) * kWarps + (threadIdx.x >> 5);
  const uint64_t nwarps = uint64_t(gridDim.x) * kWarps;
  for (uint64_t t = warp; t < batch.total_tiles; t += nwarps) {
    uint32_t lo = 0, hi = batch.n - 1;
    while (lo < hi) {
      const uint32_t mid = (lo + hi + 1) >> 1;
      if (batch.d[mid].tile_begin <= t) lo = mid; else hi = mid - 1;
    }
    const Desc& dsc = batch.d[lo];
    const uint64_t mis = dsc.dst & 127u;
    const uint64_t local = t - dsc.tile_begin;
    const uint64_t b = local == 0 ? 0 : local * kTile - mis;
    uint64_t e = (local + 1) * kTile - mis;
    if (e > dsc.len) e = dsc.len;
    copy_span(reinterpret_cast<const uint8_t*>(dsc.src) + b, reinterpret_cast<uint8_t*>(dsc.dst) + b, e - b, lane);
  }
}

int launch_gather(cudaStream_t stream, const lzk_copy_desc* d, uint32_t n, uint32_t max_ctas) {
  if (n == 0) return LZK_OK;
  if (d == nullptr) return fail(LZK_ERR_INVALID, "gather: null descriptor array");
  if (max_ctas == 0) max_ctas = 4;  // 2 saturate the host link (profiles/r02_ctasweep.jsonl)
  // Stack-allocating 31 KB is fine for host threads; keep it static per thread.
  thread_local DescBatch batch;
  uint32_t i = 0;
  while (i < n) {
    batch.n = 0;
    uint64_t tiles = 0;
    for (; i < n && batch.n < kMaxDescPerLaunch; ++i) {
      if (d[i].len == 0) continue;
      Desc& x = batch.d[batch.n++];
      x.src = d[i].src;
      x.dst = d[i].dst;
      x.len = d[i].len;
      x.tile_begin = tiles;
      tiles += (d[i].len + (d[i].dst & 127u) + kTile - 1) / kTile;
    }
    if (batch.n == 0) continue;
    batch.total_tiles = tiles;
    uint32_t grid = static_cast<uint32_t>(std::min<uint64_t>((tiles + kWarps - 1) / kWarps, max_ctas));
    lzk_gather_kernel<<<grid, kThreads, 0, stream>>>(batch);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "lzk_gather_kernel launch");
    lzk_detail::launches.fetch_add(1, std::memory_order_relaxed);
  }
  return LZK_OK;
}

// ---------------------------------------------------------------------------
// workload fill + busy compute
// ---------------------------------------------------------------------------

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void lzk_fill_kernel(uint8_t* dst, uint64_t bytes, uint64_t seed, uint64_t leaf) {
  const uint64_t base = seed ^ (leaf * 0xD1B54A32D192ED03ull);
  const uint64_t words = bytes >> 3;
  const bool aligned = (reinterpret_cast<uintptr_t>(dst) & 7u) == 0;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t w = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; w < words;
       w += stride) {
    uint64_t v = mix64(base + (w + 1) * 0x9E3779B97F4A7C15ull);
    if (aligned) {
      reinterpret_cast<uint64_t*>(dst)[w] = v;
    } else {
#pragma unroll
      for (int b = 0; b < 8; ++b) dst[w * 8 + b] = static_cast<uint8_t>(v >> (8 * b));
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && (bytes & 7u)) {
    uint64_t v = mix64(base + (words + 1) * 0x9E3779B97F4A7C15ull);
    for (uint64_t b = 0; b < (bytes & 7u); ++b) dst[words * 8 + b] = static_cast<uint8_t>(v >> (8 * b));
  }
}

__global__ void lzk_busy_kernel(float* buf, uint64_t n, uint32_t iters) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    float x = buf[i], y = 1.0001f;
    for (uint32_t k = 0; k < iters; ++k) {
      x = fmaf(x, y, 0.5f);
      y = fmaf(y, 0.9999f, 1e-7f);
    }
    buf[i] = x;
  }
}

}  // namespace

struct lzk_event {
  cudaEvent_t e = nullptr;
  int device = 0;
};

extern "C" {

const char* lzk_last_error(void) { return lzk_detail::g_err.c_str(); }

int lzk_device_count(int* count) {
  if (!count) return fail(LZK_ERR_INVALID, "null count");
  *count = 0;
  cudaError_t e = cudaGetDeviceCount(count);
  if (e != cudaSuccess) {
    *count = 0;
    return cuda_fail(e, "cudaGetDeviceCount");
  }
  return LZK_OK;
}

int lzk_set_device(int device) {
  LZK_CK(cudaSetDevice(device));
  return LZK_OK;
}

int lzk_get_device(int* device) {
  if (!device) return fail(LZK_ERR_INVALID, "null device");
  LZK_CK(cudaGetDevice(device));
  return LZK_OK;
}

uint64_t lzk_kernel_launches(void) { return lzk_detail::launches.load(); }

int lzk_dev_alloc(int device, uint64_t bytes, void** ptr) {
  if (!ptr) return fail(LZK_ERR_INVALID, "null out pointer");
  *ptr = nullptr;
  if (int rc = use_device(device)) return rc;
  LZK_CK(cudaMalloc(ptr, bytes ? bytes : 1));
  return LZK_OK;
}

int lzk_dev_free(int device, void* ptr) {
  if (!ptr) return LZK_OK;
  if (int rc = use_device(device)) return rc;
  LZK_CK(cudaFree(ptr));
  return LZK_OK;
}

int lzk_dev_memset(int device, void* ptr, int value, uint64_t bytes) {
  if (int rc = use_device(device)) return rc;
  cudaStream_t s = helper_stream(device);
  if (!s) return fail(LZK_ERR_CUDA, "helper stream");
  LZK_CK(cudaMemsetAsync(ptr, value, bytes, s));
  LZK_CK(cudaStreamSynchronize(s));
  return LZK_OK;
}

static int sync_copy(int device, void* dst, const void* src, uint64_t bytes, cudaMemcpyKind kind) {
  if (bytes == 0) return LZK_OK;
  if (int rc = use_device(device)) return rc;
  cudaStream_t s = helper_stream(device);
  if (!s) return fail(LZK_ERR_CUDA, "helper stream");
  LZK_CK(cudaMemcpyAsync(dst, src, bytes, kind, s));
  LZK_CK(cudaStreamSynchronize(s));
  return LZK_OK;
}

int lzk_memcpy_h2d(int device, void* dst, const void* src, uint64_t bytes) {
  return sync_copy(device, dst, src, bytes, cudaMemcpyHostToDevice);
}
int lzk_memcpy_d2h(int device, void* dst, const void* src, uint64_t bytes) {
  return sync_copy(device, dst, src, bytes, cudaMemcpyDeviceToHost);
}
int lzk_memcpy_d2d(int device, void* dst, const void* src, uint64_t bytes) {
  return sync_copy(device, dst, src, bytes, cudaMemcpyDeviceToDevice);
}

// ---- pinned host memory ----------------------------------------------------

namespace {
std::mutex g_host_mu;
std::unordered_map<void*, std::pair<uint64_t, bool>> g_host_allocs;  // ptr -> (bytes, mmapped)
// Released pinned blocks kept registered for reuse (engines are created and
// destroyed often in tests/harnesses; pinning dominates their cost). Bounded.
struct CachedBlock {
  void* p;
  uint64_t len;
  int flags;
};
std::vector<CachedBlock> g_host_cache;
std::unordered_map<void*, int> g_host_flags;
uint64_t g_host_cache_bytes = 0;
constexpr uint64_t kHostCacheMax = 4ull << 30;
constexpr uint64_t kHostCacheBlockMax = 1ull << 30;
}  // namespace

namespace {

// CPUs of a NUMA node, from /sys/devices/system/node/node<N>/cpulist.
bool node_cpus(int node, cpu_set_t* set) {
  std::ifstream in("/sys/devices/system/node/node" + std::to_string(node) + "/cpulist");
  std::string list;
  if (!in || !std::getline(in, list)) return false;
  CPU_ZERO(set);
  std::stringstream ss(list);
  std::string part;
  bool any = false;
  while (std::getline(ss, part, ',')) {
    const auto dash = part.find('-');
    const int a = std::stoi(part.substr(0, dash));
    const int b = dash == std::string::npos ? a : std::stoi(part.substr(dash + 1));
    for (int c = a; c <= b && c < CPU_SETSIZE; ++c) {
      CPU_SET(c, set);
      any = true;
    }
  }
  return any;
}

// Page placement policy for [p, p+len) before first touch: MPOL_PREFERRED on
// `node` (pages go there while it has memory, elsewhere rather than failing).
void prefer_node(void* p, uint64_t len, int node) {
  if (node < 0 || node >= 1024) return;
  unsigned long mask[1024 / (8 * sizeof(unsigned long))] = {};
  mask[node / (8 * sizeof(unsigned long))] = 1ul << (node % (8 * sizeof(unsigned long)));
  constexpr int kMpolPreferred = 1;
  syscall(SYS_mbind, p, len, kMpolPreferred, mask, 1024ul, 0u);
}

}  // namespace

int lzk_device_numa_node(int device, int* node) {
  if (!node) return fail(LZK_ERR_INVALID, "null out pointer");
  *node = -1;
  char bus[32] = {};
  LZK_CK(cudaDeviceGetPCIBusId(bus, sizeof bus, device));
  std::string id(bus);
  for (auto& c : id) c = char(std::tolower(static_cast<unsigned char>(c)));
  std::ifstream in("/sys/bus/pci/devices/" + id + "/numa_node");
  int n = -1;
  if (in >> n) *node = n < 0 ? -1 : n;
  return LZK_OK;
}

int lzk_host_alloc(uint64_t bytes, int flags, void** ptr) { return lzk_host_alloc_numa(bytes, flags, -1, ptr); }

int lzk_host_alloc_numa(uint64_t bytes, int flags, int numa_node, void** ptr) {
  if (!ptr) return fail(LZK_ERR_INVALID, "null out pointer");
  *ptr = nullptr;
  if (bytes == 0) bytes = 1;
  if (numa_node < -1) numa_node = -1;
  // cached blocks are matched on kind = flags + node
  const int kind = flags | ((numa_node + 1) << 8);
  // Anonymous mapping + first touch + cudaHostRegister pins ~10x faster than
  // cudaHostAlloc (measured: 0.29 s vs 3.36 s per 8 GiB on the B200 hosts).
  // LZK_HOST_HUGEPAGE asks for transparent huge pages on top.
  const uint64_t page = (flags & LZK_HOST_HUGEPAGE) ? (2ull << 20) : 4096;
  const uint64_t len = (bytes + page - 1) / page * page;
  {
    // best fit among cached blocks of the same kind, at most 2x the request
    std::lock_guard<std::mutex> lk(g_host_mu);
    size_t best = g_host_cache.size();
    for (size_t i = 0; i < g_host_cache.size(); ++i) {
      const auto& c = g_host_cache[i];
      if (c.flags == kind && c.len >= len && c.len <= 2 * len &&
          (best == g_host_cache.size() || c.len < g_host_cache[best].len)) {
        best = i;
      }
    }
    if (best < g_host_cache.size()) {
      const CachedBlock c = g_host_cache[best];
      g_host_cache.erase(g_host_cache.begin() + long(best));
      g_host_cache_bytes -= c.len;
      g_host_allocs[c.p] = {c.len, true};
      *ptr = c.p;
      return LZK_OK;
    }
  }
  void* p = mmap(nullptr, len, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  if (p == MAP_FAILED) return fail(LZK_ERR_NOMEM, "mmap of pinned memory failed");
  if (flags & LZK_HOST_HUGEPAGE) madvise(p, len, MADV_HUGEPAGE);
  // placement before the first touch: the GPU's NUMA node, touched by that
  // node's CPUs (a no-op on single-node hosts)
  cpu_set_t cpus;
  const bool bind = numa_node >= 0 && node_cpus(numa_node, &cpus);
  if (numa_node >= 0) prefer_node(p, len, numa_node);
  // first touch (page zeroing dominates pinning): parallel for big ranges
  const unsigned nt = len >= (256ull << 20) ? std::max(1u, std::min(16u, std::thread::hardware_concurrency())) : 1u;
  auto touch = [=](unsigned t) {
    if (bind) sched_setaffinity(0, sizeof cpus, &cpus);
    const uint64_t chunk = (len / nt + page - 1) / page * page;
    const uint64_t b = chunk * t, e = std::min(len, b + chunk);
    for (uint64_t o = b; o < e; o += 4096) static_cast<volatile char*>(p)[o] = 0;
  };
  if (nt == 1) {
    std::thread(touch, 0).join();  // own thread: the caller's affinity stays as it was
  } else {
    std::vector<std::thread> th;
    for (unsigned t = 0; t < nt; ++t) th.emplace_back(touch, t);
    for (auto& t : th) t.join();
  }
  const unsigned reg = cudaHostRegisterPortable | ((flags & LZK_HOST_MAPPED) ? cudaHostRegisterMapped : 0);
  const cudaError_t e = cudaHostRegister(p, len, reg);
  if (e != cudaSuccess) {
    munmap(p, len);
    return cuda_fail(e, "cudaHostRegister");
  }
  std::lock_guard<std::mutex> lk(g_host_mu);
  g_host_allocs[p] = {len, true};
  g_host_flags[p] = kind;
  *ptr = p;
  return LZK_OK;
}

int lzk_host_free(void* ptr) {
  if (!ptr) return LZK_OK;
  std::pair<uint64_t, bool> info{0, false};
  {
    std::lock_guard<std::mutex> lk(g_host_mu);
    auto it = g_host_allocs.find(ptr);
    if (it == g_host_allocs.end()) return fail(LZK_ERR_INVALID, "lzk_host_free: unknown pointer");
    info = it->second;
    g_host_allocs.erase(it);
    const int flags = g_host_flags[ptr];
    if (info.first <= kHostCacheBlockMax && g_host_cache_bytes + info.first <= kHostCacheMax) {
      g_host_cache.push_back({ptr, info.first, flags});  // stays registered for reuse
      g_host_cache_bytes += info.first;
      return LZK_OK;
    }
    g_host_flags.erase(ptr);
  }
  cudaHostUnregister(ptr);
  munmap(ptr, info.first);
  return LZK_OK;
}

int lzk_host_register(void* ptr, uint64_t bytes) {
  LZK_CK(cudaHostRegister(ptr, bytes, cudaHostRegisterPortable | cudaHostRegisterMapped));
  return LZK_OK;
}

int lzk_host_unregister(void* ptr) {
  LZK_CK(cudaHostUnregister(ptr));
  return LZK_OK;
}

// ---- streams / events --------------------------------------------------------

int lzk_stream_create(int device, int priority, lzk_stream** out) {
  if (!out) return fail(LZK_ERR_INVALID, "null out pointer");
  *out = nullptr;
  if (int rc = use_device(device)) return rc;
  int least = 0, greatest = 0;
  LZK_CK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
  // least == 0 == the default priority on current GPUs: there is nothing below
  // an ordinary stream, so priority > 0 means "no boost", not "demoted".
  int p = priority > 0 ? least : (priority < 0 ? greatest : 0);
  auto* s = new (std::nothrow) lzk_stream();
  if (!s) return fail(LZK_ERR_NOMEM, "stream");
  cudaError_t e = cudaStreamCreateWithPriority(&s->s, cudaStreamNonBlocking, p);
  if (e != cudaSuccess) {
    delete s;
    return cuda_fail(e, "cudaStreamCreateWithPriority");
  }
  s->device = device;
  *out = s;
  return LZK_OK;
}

int lzk_stream_wrap(int device, void* cuda_stream, lzk_stream** out) {
  if (!out) return fail(LZK_ERR_INVALID, "null out pointer");
  auto* s = new (std::nothrow) lzk_stream();
  if (!s) return fail(LZK_ERR_NOMEM, "stream");
  s->s = static_cast<cudaStream_t>(cuda_stream);
  s->device = device;
  s->owned = false;
  *out = s;
  return LZK_OK;
}

int lzk_stream_destroy(lzk_stream* s) {
  if (!s) return LZK_OK;
  if (s->owned && s->s) {
    use_device(s->device);
    cudaStreamSynchronize(s->s);
    cudaStreamDestroy(s->s);
  }
  delete s;
  return LZK_OK;
}

int lzk_stream_sync(lzk_stream* s) {
  if (!s) return fail(LZK_ERR_INVALID, "null stream");
  LZK_CK(cudaStreamSynchronize(s->s));
  return LZK_OK;
}

void* lzk_stream_handle(lzk_stream* s) { return s ? static_cast<void*>(s->s) : nullptr; }
int lzk_stream_device(lzk_stream* s) { return s ? s->device : -1; }

int lzk_event_create(int device, int blocking_sync, lzk_event** out) {
  if (!out) return fail(LZK_ERR_INVALID, "null out pointer");
  *out = nullptr;
  if (int rc = use_device(device)) return rc;
  auto* e = new (std::nothrow) lzk_event();
  if (!e) return fail(LZK_ERR_NOMEM, "event");
  unsigned flags = blocking_sync ? cudaEventBlockingSync : cudaEventDefault;
  cudaError_t err = cudaEventCreateWithFlags(&e->e, flags);
  if (err != cudaSuccess) {
    delete e;
    return cuda_fail(err, "cudaEventCreateWithFlags");
  }
  e->device = device;
  *out = e;
  return LZK_OK;
}

// ---- CUDA IPC (uplink relay between ranks of one node) ------------------------

namespace {

static_assert(sizeof(cudaIpcMemHandle_t) == sizeof(lzk_ipc_handle), "IPC handle size");
static_assert(sizeof(cudaIpcEventHandle_t) == sizeof(lzk_ipc_handle), "IPC handle size");

// cuMemGetAddressRange through the runtime's driver entry point: the device
// layer does not link libcuda directly (hosts without a driver still load it).
using AddressRangeFn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);

AddressRangeFn address_range() {
  static AddressRangeFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      return AddressRangeFn(nullptr);
    }
    return reinterpret_cast<AddressRangeFn>(f);
  }();
  return fn;
}

// A handle opens once per process: cache (device, handle bytes) -> base.
std::mutex g_ipc_mu;
std::vector<std::pair<std::pair<int, std::string>, void*>> g_ipc_open;

}  // namespace

int lzk_ipc_export_mem(int device, const void* dev_ptr, lzk_ipc_handle* handle, uint64_t* offset) {
  if (!dev_ptr || !handle || !offset) return fail(LZK_ERR_INVALID, "ipc export: null argument");
  if (int rc = use_device(device)) return rc;
  AddressRangeFn range = address_range();
  if (!range) return fail(LZK_ERR_CUDA, "ipc export: cuMemGetAddressRange unavailable");
  CUdeviceptr base = 0;
  size_t size = 0;
  if (range(&base, &size, reinterpret_cast<CUdeviceptr>(dev_ptr)) != CUDA_SUCCESS) {
    return fail(LZK_ERR_CUDA, "ipc export: pointer is not a device allocation");
  }
  cudaIpcMemHandle_t h;
  LZK_CK(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
  std::memcpy(handle, &h, sizeof h);
  *offset = reinterpret_cast<uint64_t>(dev_ptr) - uint64_t(base);
  return LZK_OK;
}

int lzk_ipc_open_mem(int device, const lzk_ipc_handle* handle, void** base) {
  if (!handle || !base) return fail(LZK_ERR_INVALID, "ipc open: null argument");
  if (int rc = use_device(device)) return rc;
  const std::string key(reinterpret_cast<const char*>(handle), sizeof *handle);
  std::lock_guard<std::mutex> lk(g_ipc_mu);
  for (const auto& [k, p] : g_ipc_open) {
    if (k.first == device && k.second == key) {
      *base = p;
      return LZK_OK;
    }
  }
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof h);
  void* p = nullptr;
  LZK_CK(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
  g_ipc_open.push_back({{device, key}, p});
  *base = p;
  return LZK_OK;
}

int lzk_ipc_close_all(void) {
  std::lock_guard<std::mutex> lk(g_ipc_mu);
  for (const auto& [k, p] : g_ipc_open) {
    use_device(k.first);
    cudaIpcCloseMemHandle(p);
  }
  g_ipc_open.clear();
  return LZK_OK;
}

int lzk_ipc_event_create(int device, lzk_event** out, lzk_ipc_handle* handle) {
  if (!out || !handle) return fail(LZK_ERR_INVALID, "ipc event: null argument");
  *out = nullptr;
  if (int rc = use_device(device)) return rc;
  auto* e = new (std::nothrow) lzk_event();
  if (!e) return fail(LZK_ERR_NOMEM, "event");
  cudaError_t err = cudaEventCreateWithFlags(&e->e, cudaEventDisableTiming | cudaEventInterprocess);
  cudaIpcEventHandle_t h;
  if (err == cudaSuccess) err = cudaIpcGetEventHandle(&h, e->e);
  if (err != cudaSuccess) {
    if (e->e) cudaEventDestroy(e->e);
    delete e;
    return cuda_fail(err, "interprocess event");
  }
  std::memcpy(handle, &h, sizeof h);
  e->device = device;
  *out = e;
  return LZK_OK;
}

int lzk_ipc_event_open(int device, const lzk_ipc_handle* handle, lzk_event** out) {
  if (!out || !handle) return fail(LZK_ERR_INVALID, "ipc event open: null argument");
  *out = nullptr;
  if (int rc = use_device(device)) return rc;
  auto* e = new (std::nothrow) lzk_event();
  if (!e) return fail(LZK_ERR_NOMEM, "event");
  cudaIpcEventHandle_t h;
  std::memcpy(&h, handle, sizeof h);
  cudaError_t err = cudaIpcOpenEventHandle(&e->e, h);
  if (err != cudaSuccess) {
    delete e;
    return cuda_fail(err, "cudaIpcOpenEventHandle");
  }
  e->device = device;
  *out = e;
  return LZK_OK;
}

int lzk_event_destroy(lzk_event* e) {
  if (!e) return LZK_OK;
  use_device(e->device);
  cudaEventDestroy(e->e);
  delete e;
  return LZK_OK;
}

int lzk_event_record(lzk_event* e, lzk_stream* s) {
  if (!e || !s) return fail(LZK_ERR_INVALID, "null event/stream");
  if (int rc = use_device(s->device)) return rc;
  LZK_CK(cudaEventRecord(e->e, s->s));
  return LZK_OK;
}

int lzk_event_query(lzk_event* e) {
  if (!e) return fail(LZK_ERR_INVALID, "null event");
  cudaError_t r = cudaEventQuery(e->e);
  if (r == cudaSuccess) return LZK_OK;
  if (r == cudaErrorNotReady) {
    cudaGetLastError();
    return LZK_PENDING;
  }
  return cuda_fail(r, "cudaEventQuery");
}

int lzk_event_sync(lzk_event* e) {
  if (!e) return fail(LZK_ERR_INVALID, "null event");
  LZK_CK(cudaEventSynchronize(e->e));
  return LZK_OK;
}

int lzk_event_elapsed_ms(lzk_event* a, lzk_event* b, float* ms) {
  if (!a || !b || !ms) return fail(LZK_ERR_INVALID, "null arg");
  LZK_CK(cudaEventElapsedTime(ms, a->e, b->e));
  return LZK_OK;
}

int lzk_stream_wait_event(lzk_stream* s, lzk_event* e) {
  if (!s || !e) return fail(LZK_ERR_INVALID, "null stream/event");
  LZK_CK(cudaStreamWaitEvent(s->s, e->e, 0));
  return LZK_OK;
}

int lzk_event_record_raw(lzk_event* e, void* cuda_stream) {
  if (!e) return fail(LZK_ERR_INVALID, "null event");
  if (int rc = use_device(e->device)) return rc;
  LZK_CK(cudaEventRecord(e->e, static_cast<cudaStream_t>(cuda_stream)));
  return LZK_OK;
}

int lzk_stream_wait_raw(lzk_stream* s, void* producer_stream) {
  if (!s) return fail(LZK_ERR_INVALID, "null stream");
  if (int rc = use_device(s->device)) return rc;
  cudaEvent_t e = nullptr;
  LZK_CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  cudaError_t r = cudaEventRecord(e, static_cast<cudaStream_t>(producer_stream));
  if (r == cudaSuccess) r = cudaStreamWaitEvent(s->s, e, 0);
  cudaEventDestroy(e);  // released once the queued wait has fired
  if (r != cudaSuccess) return cuda_fail(r, "lzk_stream_wait_raw");
  return LZK_OK;
}

int lzk_raw_stream_wait_event(void* cuda_stream, lzk_event* e) {
  if (!e) return fail(LZK_ERR_INVALID, "null event");
  LZK_CK(cudaStreamWaitEvent(static_cast<cudaStream_t>(cuda_stream), e->e, 0));
  return LZK_OK;
}

// ---- copies ------------------------------------------------------------------

int lzk_gather_d2h(lzk_stream* s, const lzk_copy_desc* d, uint32_t n, uint32_t max_ctas) {
  if (!s) return fail(LZK_ERR_INVALID, "null stream");
  if (int rc = use_device(s->device)) return rc;
  return launch_gather(s->s, d, n, max_ctas);
}

int lzk_scatter_h2d(lzk_stream* s, const lzk_copy_desc* d, uint32_t n, uint32_t max_ctas) {
  if (!s) return fail(LZK_ERR_INVALID, "null stream");
  if (int rc = use_device(s->device)) return rc;
  // Reads over PCIe have ~us latency: use a wider grid to keep enough loads
  // in flight.
  return launch_gather(s->s, d, n, max_ctas ? max_ctas : 64);
}

int lzk_gather_d2d(lzk_stream* s, const lzk_copy_desc* d, uint32_t n, uint32_t max_ctas) {
  if (!s) return fail(LZK_ERR_INVALID, "null stream");
  if (int rc = use_device(s->device)) return rc;
  return launch_gather(s->s, d, n, max_ctas ? max_ctas : 296);
}

static int ce_copy(lzk_stream* s, const lzk_copy_desc* d, uint32_t n, cudaMemcpyKind kind) {
  if (!s) return fail(LZK_ERR_INVALID, "null stream");
  if (n && !d) return fail(LZK_ERR_INVALID, "null descriptor array");
  if (int rc = use_device(s->device)) return rc;
  for (uint32_t i = 0; i < n; ++i) {
    if (d[i].len == 0) continue;
    LZK_CK(cudaMemcpyAsync(reinterpret_cast<void*>(d[i].dst), reinterpret_cast<const void*>(d[i].src),
                           d[i].len, kind, s->s));
  }
  return LZK_OK;
}

int lzk_ce_copy_d2h(lzk_stream* s, const lzk_copy_desc* d, uint32_t n) {
  return ce_copy(s, d, n, cudaMemcpyDeviceToHost);
}

int lzk_ce_copy_h2d(lzk_stream* s, const lzk_copy_desc* d, uint32_t n) {
  return ce_copy(s, d, n, cudaMemcpyHostToDevice);
}

int lzk_ce_copy_d2d(lzk_stream* s, const lzk_copy_desc* d, uint32_t n) {
  return ce_copy(s, d, n, cudaMemcpyDeviceToDevice);
}

int lzk_fill_splitmix(lzk_stream* s, void* dev, uint64_t bytes, uint64_t seed, uint64_t leaf) {
  if (!s) return fail(LZK_ERR_INVALID, "null stream");
  if (bytes == 0) return LZK_OK;
  if (int rc = use_device(s->device)) return rc;
  uint64_t words = (bytes >> 3) + 1;
  uint32_t grid = static_cast<uint32_t>(std::min<uint64_t>((words + 255) / 256, 148ull * 8));
  lzk_fill_kernel<<<grid, 256, 0, s->s>>>(static_cast<uint8_t*>(dev), bytes, seed, leaf);
  LZK_CK(cudaGetLastError());
  lzk_detail::launches.fetch_add(1, std::memory_order_relaxed);
  return LZK_OK;
}

void lzk_range_push(const char* name) { nvtxRangePushA(name ? name : "lzk"); }
void lzk_range_pop(void) { nvtxRangePop(); }

int lzk_busy_compute(lzk_stream* s, float* buf, uint64_t n, uint32_t iters, uint32_t ctas) {
  if (!s) return fail(LZK_ERR_INVALID, "null stream");
  if (int rc = use_device(s->device)) return rc;
  lzk_busy_kernel<<<ctas ? ctas : 148 * 4, 256, 0, s->s>>>(buf, n, iters);
  LZK_CK(cudaGetLastError());
  lzk_detail::launches.fetch_add(1, std::memory_order_relaxed);
  return LZK_OK;
}

}  // extern "C"
