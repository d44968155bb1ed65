// B200 (sm_100a) FNV-1a-64 over many device byte ranges.
//
// The reference checksums every shard entry on the host, byte-serially
// (include/lzckpt/checksum.hpp:17-24; folded per chunk in
// src/flush_pipeline.cpp:194-263 and re-computed by the restore check in
// src/format.cpp:173-214). One core folds ~0.7 GB/s, and the B200 hosts have
// 16 cores for 8 GPUs that each snapshot at ~57 GB/s. This file computes the
// same digests on the device, bit-exactly.
//
// Algorithm (executable model: tools/fnv_scan_model.py)
//  * Step h' = (h ^ b) * P, P = 2^40 + 0x1b3. The low byte l = h & 0xff
//    evolves on its own: l' = 0xb3 * (l ^ b) mod 256.
//  * A 64-bit state whose low byte is right follows the true trajectory's
//    low bytes, so plain FNV started from the value l gives
//    acc = P^n * l + S, and the true state is h_end = P^n * h + (acc - P^n * l).
//    A lane can therefore hash its own bytes independently once it knows the
//    low byte at their start.
//  * Those low bytes come from a bit-sliced scan. Multiplying by an odd
//    constant is a T-function: bit i of 0xb3 * x is x_i xor a function of
//    x_0..x_{i-1}. So plane i of the low-byte trajectory is a prefix-XOR of
//    known bits once planes 0..i-1 are resolved. Each lane transposes its 32
//    bytes into 8 bit-plane words. Per plane it runs an in-register prefix XOR
//    (5 shift/xor steps), then a warp ballot + popc carries the parity across
//    lanes and across 1 KiB windows. The column adder of y = x + 2x + 16x +
//    32x + 128x supplies the lower-plane terms with a few LOP3s.
//  * Per lane, two 16-byte FNV chains (low bytes at lane offsets 0 and 16)
//    run interleaved. Lane results fold as R = R * P^1024 + window sum, and
//    at the end h = P^(1024 C) h0 + sum_j R_j P^(32 (31 - j)).
//
// Two schedules:
//  * short ranges: one warp per range (largest first, round-robin), one pass;
//    about 16 integer ops per byte;
//  * long ranges (more than a fair share of the grid, >= 4 MiB): split into
//    up to 2048 segments of >= 256 KiB, all processed in parallel. Bit i of
//    a segment's outgoing low byte depends only on incoming bits <= i, so
//    plane parities can be resolved from the bottom up. Dual pass K
//    (K = 0..3) takes the carry-in bits < 2K from the XOR of the earlier
//    segments' parities and yields every segment's plane-2K parity and its
//    plane-(2K+1) parity under both values of incoming bit 2K (a flipped
//    bit 2K complements the whole x_{2K} plane); a one-warp-per-range
//    resolve kernel then picks the right hypothesis in segment order. A
//    final pass hashes every segment from its now-known incoming low byte,
//    and one warp per range folds the segments affinely (h = P^len h + S).
//    Four dual passes do 24 plane scans per window where eight single-plane
//    passes did 36 (tools/fnv_scan_model.py models both schedules).
#include <algorithm>
#include <cstdint>
#include <mutex>
#include <numeric>
#include <vector>

#include "lzk_internal.h"

namespace {

using lzk_detail::cuda_fail;
using lzk_detail::fail;
using lzk_detail::use_device;

constexpr uint64_t kPrime = 0x100000001b3ull;
// Two CTA shapes, same 32 resident warps per SM at 64 registers:
//  * short ranges only (one warp per range): 128-thread CTAs, 8 per SM, so the
//    block scheduler spreads the warps evenly (512-thread CTAs put 4096 ranges
//    on 108 SMs with 32 warps and 40 with 16: uniform 1 MiB ranges 1.26 ->
//    1.33 TB/s);
//  * batches with segmented long ranges: 512-thread CTAs, 2 per SM (their
//    multi-pass schedule measured ~9 % faster that way).
// The C ABI's max_ctas counts 512-thread CTA equivalents (about one SM each).
constexpr int kBigThreads = 512;
constexpr int kSmallThreads = 128;
constexpr uint32_t kWarpsPerSm = 32;
constexpr int kHashWarps = kBigThreads / 32;  // warps per max_ctas unit
constexpr uint64_t kSegMin = 256ull << 10;  // bytes, multiple of 1 KiB
constexpr uint32_t kMaxSegs = 2048;         // per range
constexpr uint64_t kLongMin = 4ull << 20;

constexpr uint64_t cpow(uint64_t b, uint64_t e) {
  uint64_t r = 1;
  while (e) {
    if (e & 1) r *= b;
    b *= b;
    e >>= 1;
  }
  return r;
}
constexpr uint64_t kP16 = cpow(kPrime, 16);
constexpr uint64_t kP1024 = cpow(kPrime, 1024);

struct HashItem {
  lzk_hash_desc d;
  uint32_t seg_begin;  // exclusive prefix of nseg over the batch
  uint32_t nseg;       // 1 = short range (one warp, one pass)
  uint64_t seglen;     // segment body bytes (multiple of 1 KiB) when nseg > 1
};

// The item table lives in device memory (any number of ranges per launch).
struct HashBatch {
  const HashItem* it;
  uint32_t n;
  uint32_t pad0;
  uint32_t total_segs;
  uint32_t pad;
};

__device__ __forceinline__ uint64_t pow64(uint64_t b, uint64_t e) {
  uint64_t r = 1;
  while (e) {
    if (e & 1) r *= b;
    b *= b;
    e >>= 1;
  }
  return r;
}

__device__ __forceinline__ uint4 ld_nc(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// w >> (32 - k) as IMAD.HI on the FMA pipe (the kernel is bound by the ALU
// pipe, where SHF would go).
__device__ __forceinline__ uint32_t hi_shift(uint32_t w, uint32_t two_k) {
  uint32_t r;
  asm("mul.hi.u32 %0, %1, %2;" : "=r"(r) : "r"(w), "r"(two_k));
  return r;
}

__device__ __forceinline__ uint64_t fnv_word(uint64_t h, uint32_t w) {
  h = (h ^ (w & 0xffu)) * kPrime;
  h = (h ^ (hi_shift(w, 1u << 24) & 0xffu)) * kPrime;
  h = (h ^ (hi_shift(w, 1u << 16) & 0xffu)) * kPrime;
  h = (h ^ hi_shift(w, 1u << 8)) * kPrime;
  return h;
}

__device__ __forceinline__ uint32_t maj3(uint32_t a, uint32_t b, uint32_t c) {
  return (a & b) | (a & c) | (b & c);
}

// o[t] = byte t of a, b, c, d (a 4x4 byte transpose in 8 PRMTs).
__device__ __forceinline__ void bytes4x4(uint32_t a, uint32_t b, uint32_t c, uint32_t d, uint32_t* o) {
  const uint32_t ab_lo = __byte_perm(a, b, 0x5140), ab_hi = __byte_perm(a, b, 0x7362);
  const uint32_t cd_lo = __byte_perm(c, d, 0x5140), cd_hi = __byte_perm(c, d, 0x7362);
  o[0] = __byte_perm(ab_lo, cd_lo, 0x5410);
  o[1] = __byte_perm(ab_lo, cd_lo, 0x7632);
  o[2] = __byte_perm(ab_hi, cd_hi, 0x5410);
  o[3] = __byte_perm(ab_hi, cd_hi, 0x7632);
}

__device__ __forceinline__ void delta_swap(uint32_t& a, uint32_t& b, uint32_t mask, int s) {
  const uint32_t x = ((a >> s) ^ b) & mask;
  b ^= x;
  a ^= x << s;
}

// 32 bytes (w[q] holds bytes 4q..4q+3, little endian) -> 8 bit planes,
// bit p of B[i] = bit i of byte p. A byte shuffle puts byte 8k+t in byte k
// of word t, then three delta-swap stages transpose each byte lane's 8x8 bit
// matrix across the eight words.
__device__ __forceinline__ void to_planes(const uint32_t* w, uint32_t* B) {
  bytes4x4(w[0], w[2], w[4], w[6], B);
  bytes4x4(w[1], w[3], w[5], w[7], B + 4);
#pragma unroll
  for (int t = 0; t < 4; ++t) delta_swap(B[t], B[t + 4], 0x0f0f0f0fu, 4);
  delta_swap(B[0], B[2], 0x33333333u, 2);
  delta_swap(B[1], B[3], 0x33333333u, 2);
  delta_swap(B[4], B[6], 0x33333333u, 2);
  delta_swap(B[5], B[7], 0x33333333u, 2);
#pragma unroll
  for (int t = 0; t < 8; t += 2) delta_swap(B[t], B[t + 1], 0x55555555u, 1);
}

// Low bytes of one warp window: lane j holds bytes [32j, 32j + 32) in w.
// Resolves planes 0..NP-1. `carry[i]` (warp-uniform, 0 or 1) is bit i of the
// low byte at the window start and is advanced past it. `valid` masks the
// lane's positions that exist (partial last window). Outputs the low bytes
// at the lane's offsets 0 and 16 (meaningful when NP == 8). The kernel is
// bound by the ALU pipe, so bit bookkeeping uses multiplies (FMA pipe) and the
// carries stay unpacked.
template <int NP>
__device__ __forceinline__ void scan_planes(const uint32_t* w, uint32_t* carry, uint32_t lt, uint32_t valid,
                                            uint32_t& l0, uint32_t& l16) {
  uint32_t B[8];
  to_planes(w, B);
  uint32_t lstart = 0, q = 0;
  // plane i: l_i at each position = carry-in xor exclusive prefix-XOR of
  // e_i; returns x_i = l_i ^ b_i. Bit 16 of l_i is bit 15 of the prefix
  // xor the carry-in, so the offset-16 low byte is lstart ^ (q >> 15).
  auto plane = [&](int i, uint32_t e) -> uint32_t {
    uint32_t p = e & valid;
    p ^= p << 1;
    p ^= p << 2;
    p ^= p << 4;
    p ^= p << 8;
    p ^= p << 16;
    const uint32_t bal = __ballot_sync(0xffffffffu, p >> 31);
    const uint32_t cin = (__popc(bal & lt) ^ carry[i]) & 1u;
    carry[i] ^= __popc(bal) & 1u;
    lstart += cin * (1u << i);
    q += (p & 0x8000u) * (1u << i);
    return (p << 1) ^ (cin * 0xffffffffu) ^ B[i];
  };
  // column adder of y = 179 x (mod 256): column i sums x_i, x_{i-1},
  // x_{i-4}, x_{i-5}, x_{i-7} and the carries from column i-1.
  const uint32_t x0 = plane(0, B[0]);
  if constexpr (NP > 1) {
    const uint32_t x1 = plane(1, B[1] ^ x0);
    const uint32_t c2 = x1 & x0;
    if constexpr (NP > 2) {
      const uint32_t x2 = plane(2, B[2] ^ x1 ^ c2);
      const uint32_t c3 = maj3(x2, x1, c2);
      if constexpr (NP > 3) {
        const uint32_t x3 = plane(3, B[3] ^ x2 ^ c3);
        const uint32_t c4 = maj3(x3, x2, c3);
        if constexpr (NP > 4) {
          const uint32_t x4 = plane(4, B[4] ^ x3 ^ x0 ^ c4);
          const uint32_t k1 = maj3(x4, x3, x0), k2 = (x4 ^ x3 ^ x0) & c4;
          if constexpr (NP > 5) {
            const uint32_t x5 = plane(5, B[5] ^ x4 ^ x1 ^ x0 ^ k1 ^ k2);
            const uint32_t s1 = x5 ^ x4 ^ x1, m1 = maj3(x5, x4, x1);
            const uint32_t s2 = x0 ^ k1 ^ k2, m2 = maj3(x0, k1, k2);
            const uint32_t m3 = s1 & s2;
            if constexpr (NP > 6) {
              const uint32_t x6 = plane(6, B[6] ^ x5 ^ x2 ^ x1 ^ m1 ^ m2 ^ m3);
              const uint32_t t1 = x6 ^ x5 ^ x2, n1 = maj3(x6, x5, x2);
              const uint32_t t2 = x1 ^ m1 ^ m2, n2 = maj3(x1, m1, m2);
              const uint32_t n3 = maj3(m3, t1, t2);
              if constexpr (NP > 7) plane(7, B[7] ^ x6 ^ x3 ^ x2 ^ x0 ^ n1 ^ n2 ^ n3);
            }
          }
        }
      }
    }
  }
  l0 = lstart;
  l16 = lstart ^ (q >> 15);
}

__device__ __forceinline__ uint64_t warp_sum(uint64_t v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ uint32_t head_len(uint64_t src, uint64_t len) {
  const uint64_t h = (16u - (src & 15u)) & 15u;
  return static_cast<uint32_t>(h < len ? h : len);
}

__device__ __forceinline__ uint64_t fold_bytes(uint64_t h, const uint8_t* p, uint32_t n) {
  for (uint32_t i = 0; i < n; ++i) h = (h ^ p[i]) * kPrime;
  return h;
}

// FNV-1a-64 of n bytes at p continuing from state h; all 32 lanes call it
// with the same arguments and get the same result.
__device__ uint64_t hash_range(const uint8_t* p, uint64_t n, uint64_t h, uint32_t lane, uint32_t lt,
                               uint64_t wlane) {
  const uint32_t head = head_len(reinterpret_cast<uintptr_t>(p), n);
  h = fold_bytes(h, p, head);  // every lane, redundantly
  p += head;
  n -= head;

  uint32_t carry[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) carry[i] = (static_cast<uint32_t>(h) >> i) & 1u;
  const uint64_t windows = n >> 10;
  if (windows) {
    const uint4* q = reinterpret_cast<const uint4*>(p) + 2 * lane;
    uint4 a = ld_nc(q), b = ld_nc(q + 1);
    uint64_t R = 0;
    for (uint64_t c = 0; c < windows; ++c) {
      const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
      if (c + 1 < windows) {  // prefetch the next window
        q += 64;
        a = ld_nc(q);
        b = ld_nc(q + 1);
      }
      uint32_t l0, l16;
      scan_planes<8>(w, carry, lt, 0xffffffffu, l0, l16);
      uint64_t a0 = l0, a1 = l16;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        a0 = fnv_word(a0, w[k]);
        a1 = fnv_word(a1, w[k + 4]);
      }
      R = R * kP1024 + ((a0 - kP16 * l0) * kP16 + (a1 - kP16 * l16));
    }
    h = pow64(kP1024, windows) * h + warp_sum(R * wlane);
  }

  const uint32_t rem = static_cast<uint32_t>(n & 1023u);
  if (rem) {
    const uint8_t* t = p + (windows << 10) + 32u * lane;
    const uint32_t cnt = rem > 32u * lane ? min(32u, rem - 32u * lane) : 0u;
    uint32_t w[8];
    if (cnt == 32) {
      const uint4 a = ld_nc(reinterpret_cast<const uint4*>(t)), b = ld_nc(reinterpret_cast<const uint4*>(t) + 1);
      w[0] = a.x; w[1] = a.y; w[2] = a.z; w[3] = a.w;
      w[4] = b.x; w[5] = b.y; w[6] = b.z; w[7] = b.w;
    } else {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        uint32_t v = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (uint32_t(4 * k + j) < cnt) v |= uint32_t(t[4 * k + j]) << (8 * j);
        }
        w[k] = v;
      }
    }
    uint32_t l0, l16;
    scan_planes<8>(w, carry, lt, cnt >= 32 ? 0xffffffffu : ((1u << cnt) - 1u), l0, l16);
    uint64_t acc = l0;
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      if (uint32_t(k) < cnt) acc = (acc ^ ((w[k >> 2] >> (8 * (k & 3))) & 0xffu)) * kPrime;
    }
    uint64_t v = 0;
    if (cnt) v = (acc - pow64(kPrime, cnt) * l0) * pow64(kPrime, rem - 32u * lane - cnt);
    h = pow64(kPrime, rem) * h + warp_sum(v);
  }
  return h;
}

struct Scratch {
  uint8_t* par;  // per segment: bit i = plane-i parity of the segment
  uint64_t* S;   // per segment: true state after segment 0 / relative sum of the others
  uint8_t* alt;  // per segment: bit 2K+1 = plane-(2K+1) parity if incoming bit 2K were 1
};

__device__ __forceinline__ uint32_t find_item(const HashBatch& b, uint32_t t) {
  uint32_t lo = 0, hi = b.n - 1;
  while (lo < hi) {
    const uint32_t mid = (lo + hi + 1) >> 1;
    if (b.it[mid].seg_begin <= t) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// Items reach the device through kernel parameters: each upload launch
// carries up to kUploadItems of them and writes them into the device table
// (no pinned staging, no host-side allocation per call). In continue mode
// the running state is read from *out (often mapped host memory) here, once
// per item, so no hashing warp ever reads its seed across PCIe.
constexpr uint32_t kUploadItems = 600;
struct UploadParams {
  HashItem* dst;
  uint32_t n;
  uint32_t cont;
  HashItem items[kUploadItems];
};
static_assert(sizeof(UploadParams) <= 31 * 1024, "kernel parameter budget");

__global__ void lzk_fnv_upload_kernel(const __grid_constant__ UploadParams p) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= p.n) return;
  HashItem it = p.items[i];
  if (p.cont) asm volatile("ld.volatile.u64 %0, [%1];" : "=l"(it.d.seed) : "l"(it.d.out));
  p.dst[i] = it;
}

// XOR of the parity bytes of segments [base, base + s): the low-byte
// changes accumulated before segment s.
__device__ __forceinline__ uint32_t parity_prefix(const uint8_t* par, uint32_t base, uint32_t s, uint32_t lane) {
  uint32_t x = 0;
  for (uint32_t k = lane; k < s; k += 32) x ^= par[base + k];
#pragma unroll
  for (int o = 16; o; o >>= 1) x ^= __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

__device__ __forceinline__ uint32_t prefix_xor(uint32_t p) {
  p ^= p << 1;
  p ^= p << 2;
  p ^= p << 4;
  p ^= p << 8;
  p ^= p << 16;
  return p;
}

// One full window of a dual pass: planes 0..2K resolved as in scan_planes
// (carry-ins from `carry`), then plane 2K+1's parity for BOTH values of the
// plane-2K carry-in, which this pass does not know yet. A different incoming
// bit 2K flips the whole x_{2K} plane (x = l ^ b, and l_{2K} = carry ^ prefix),
// so the second hypothesis is the column adder evaluated on ~x_{2K}. A plane's
// parity does not depend on its own carry-in, so carry[2K+1] (hypothesis 0)
// and `alt` (hypothesis 1) both start at 0.
template <int K>
__device__ __forceinline__ void scan_dual(const uint32_t* w, uint32_t* carry, uint32_t& alt, uint32_t lt) {
  uint32_t B[8];
  to_planes(w, B);
  auto plane = [&](int i, uint32_t e) -> uint32_t {
    const uint32_t p = prefix_xor(e);
    const uint32_t bal = __ballot_sync(0xffffffffu, p >> 31);
    const uint32_t cin = (__popc(bal & lt) ^ carry[i]) & 1u;
    carry[i] ^= __popc(bal) & 1u;
    return (p << 1) ^ (cin * 0xffffffffu) ^ B[i];
  };
  auto parity = [&](uint32_t e, uint32_t& c) {
    c ^= __popc(__ballot_sync(0xffffffffu, prefix_xor(e) >> 31)) & 1u;
  };
  const uint32_t x0 = plane(0, B[0]);
  if constexpr (K == 0) {
    parity(B[1] ^ x0, carry[1]);
    parity(B[1] ^ ~x0, alt);
    return;
  }
  const uint32_t x1 = plane(1, B[1] ^ x0);
  const uint32_t c2 = x1 & x0;
  const uint32_t x2 = plane(2, B[2] ^ x1 ^ c2);
  if constexpr (K == 1) {
    auto e3 = [&](uint32_t x) { return B[3] ^ x ^ maj3(x, x1, c2); };
    parity(e3(x2), carry[3]);
    parity(e3(~x2), alt);
    return;
  }
  const uint32_t c3 = maj3(x2, x1, c2);
  const uint32_t x3 = plane(3, B[3] ^ x2 ^ c3);
  const uint32_t c4 = maj3(x3, x2, c3);
  const uint32_t x4 = plane(4, B[4] ^ x3 ^ x0 ^ c4);
  auto e5 = [&](uint32_t x) { return B[5] ^ x ^ x1 ^ x0 ^ maj3(x, x3, x0) ^ ((x ^ x3 ^ x0) & c4); };
  if constexpr (K == 2) {
    parity(e5(x4), carry[5]);
    parity(e5(~x4), alt);
    return;
  }
  const uint32_t k1 = maj3(x4, x3, x0), k2 = (x4 ^ x3 ^ x0) & c4;
  const uint32_t x5 = plane(5, e5(x4));
  const uint32_t s1 = x5 ^ x4 ^ x1, m1 = maj3(x5, x4, x1);
  const uint32_t s2 = x0 ^ k1 ^ k2, m2 = maj3(x0, k1, k2);
  const uint32_t m3 = s1 & s2;
  const uint32_t x6 = plane(6, B[6] ^ x5 ^ x2 ^ x1 ^ m1 ^ m2 ^ m3);
  const uint32_t t2 = x1 ^ m1 ^ m2, n2 = maj3(x1, m1, m2);
  auto e7 = [&](uint32_t x) {
    const uint32_t t1 = x ^ x5 ^ x2;
    return B[7] ^ x ^ x3 ^ x2 ^ x0 ^ maj3(x, x5, x2) ^ n2 ^ maj3(m3, t1, t2);
  };
  parity(e7(x6), carry[7]);
  parity(e7(~x6), alt);
}

// Dual pass K of the long-range schedule (four instead of eight passes): for
// every segment with a successor, the plane-2K parity and the plane-(2K+1)
// parity under both values of the still-unknown incoming bit 2K.
template <int K>
__global__ void __launch_bounds__(kBigThreads) lzk_fnv_dual_pass_kernel(const HashBatch batch, Scratch sc) {
  constexpr uint32_t kWarps = kBigThreads / 32;
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t lt = (1u << lane) - 1u;
  const uint32_t nwarps = gridDim.x * kWarps;
  for (uint32_t t = blockIdx.x * kWarps + (threadIdx.x >> 5); t < batch.total_segs; t += nwarps) {
    const HashItem it = batch.it[find_item(batch, t)];
    const uint32_t s = t - it.seg_begin;
    if (s + 1 >= it.nseg) continue;  // nobody consumes the last segment's parities
    const uint8_t* src = reinterpret_cast<const uint8_t*>(it.d.src);
    const uint32_t head = head_len(it.d.src, it.d.len);
    const uint64_t hh = fold_bytes(it.d.seed, src, head);
    const uint32_t cin =
        (static_cast<uint32_t>(hh) ^ parity_prefix(sc.par, it.seg_begin, s, lane)) & ((1u << (2 * K)) - 1u);
    uint32_t carry[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) carry[i] = (cin >> i) & 1u;  // bits 2K and 2K+1 start at 0
    uint32_t alt = 0;
    const uint4* q = reinterpret_cast<const uint4*>(src + head + uint64_t(s) * it.seglen) + 2 * lane;
    const uint64_t windows = it.seglen >> 10;
    uint4 a = ld_nc(q), b = ld_nc(q + 1);
    for (uint64_t c = 0; c < windows; ++c) {
      const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
      if (c + 1 < windows) {
        q += 64;
        a = ld_nc(q);
        b = ld_nc(q + 1);
      }
      scan_dual<K>(w, carry, alt, lt);
    }
    if (lane == 0) {
      sc.par[t] |= static_cast<uint8_t>((carry[2 * K] << (2 * K)) | (carry[2 * K + 1] << (2 * K + 1)));
      sc.alt[t] |= static_cast<uint8_t>(alt << (2 * K + 1));
    }
  }
}

// After dual pass K: walk each long range's segments in order (32 at a time,
// ballot prefix), learn every segment's incoming bit 2K from the plane-2K
// parities, and keep the matching plane-(2K+1) hypothesis in `par`. One warp
// per range.
template <int K>
__global__ void lzk_fnv_resolve_kernel(const HashBatch batch, Scratch sc) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t lt = (1u << lane) - 1u;
  const uint32_t nwarps = gridDim.x * (blockDim.x >> 5);
  for (uint32_t i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < batch.n; i += nwarps) {
    const HashItem it = batch.it[i];
    if (it.nseg == 1) continue;
    const uint8_t* src = reinterpret_cast<const uint8_t*>(it.d.src);
    uint32_t bit = (static_cast<uint32_t>(fold_bytes(it.d.seed, src, head_len(it.d.src, it.d.len))) >> (2 * K)) & 1u;
    for (uint32_t base = 0; base + 1 < it.nseg; base += 32) {
      const uint32_t s = base + lane;
      const bool mine = s + 1 < it.nseg;
      const uint32_t p = mine ? sc.par[it.seg_begin + s] : 0u;
      const uint32_t bal = __ballot_sync(0xffffffffu, (p >> (2 * K)) & 1u);
      const uint32_t in = bit ^ (__popc(bal & lt) & 1u);  // incoming bit 2K of segment s
      if (mine && in) {
        const uint32_t hi = (sc.alt[it.seg_begin + s] >> (2 * K + 1)) & 1u;
        sc.par[it.seg_begin + s] = static_cast<uint8_t>((p & ~(1u << (2 * K + 1))) | (hi << (2 * K + 1)));
      }
      bit ^= __popc(bal) & 1u;
    }
  }
}

// Final pass: short ranges are hashed whole (result stored to out); every
// segment of a long range is hashed from its incoming low byte.
template <int T>
__global__ void __launch_bounds__(T, kWarpsPerSm * 32 / T) lzk_fnv_kernel(const HashBatch batch, Scratch sc) {
  constexpr uint32_t kWarps = T / 32;
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t lt = (1u << lane) - 1u;
  const uint32_t nwarps = gridDim.x * kWarps;
  const uint64_t wlane = pow64(kPrime, 32u * (31u - lane));
  for (uint32_t t = blockIdx.x * kWarps + (threadIdx.x >> 5); t < batch.total_segs; t += nwarps) {
    const HashItem it = batch.it[find_item(batch, t)];
    const uint32_t s = t - it.seg_begin;
    const uint8_t* src = reinterpret_cast<const uint8_t*>(it.d.src);
    const uint64_t h0 = it.d.seed;
    if (it.nseg == 1) {
      const uint64_t h = hash_range(src, it.d.len, h0, lane, lt, wlane);
      if (lane == 0) *reinterpret_cast<uint64_t*>(it.d.out) = h;
      continue;
    }
    const uint32_t head = head_len(it.d.src, it.d.len);
    if (s == 0) {
      const uint64_t h = hash_range(src, head + it.seglen, h0, lane, lt, wlane);
      if (lane == 0) sc.S[t] = h;
      continue;
    }
    const uint64_t off = head + uint64_t(s) * it.seglen;
    const uint64_t n = min(it.seglen, it.d.len - off);
    const uint32_t lin =
        (static_cast<uint32_t>(fold_bytes(h0, src, head)) ^ parity_prefix(sc.par, it.seg_begin, s, lane)) & 0xffu;
    const uint64_t acc = hash_range(src + off, n, lin, lane, lt, wlane);
    if (lane == 0) sc.S[t] = acc - pow64(kPrime, n) * lin;
  }
}

// h = S_0, then h = P^len_s * h + S_s over the remaining segments. Every
// segment is an affine map h -> M h + A (segment 0: M = 0, A = S_0); a lane
// composes a contiguous block of segments, then a shuffle-down tree composes
// the 32 block maps in order (the composition is associative, not
// commutative). One warp per long range.
__global__ void lzk_fnv_combine_kernel(const HashBatch batch, Scratch sc) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t nwarps = gridDim.x * (blockDim.x >> 5);
  for (uint32_t i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < batch.n; i += nwarps) {
    const HashItem it = batch.it[i];
    if (it.nseg == 1) continue;
    const uint64_t head = head_len(it.d.src, it.d.len);
    const uint64_t last = it.d.len - head - uint64_t(it.nseg - 1) * it.seglen;
    const uint64_t pseg = pow64(kPrime, it.seglen), plast = pow64(kPrime, last);
    const uint32_t per = (it.nseg + 31u) / 32u;
    const uint32_t b0 = min(it.nseg, lane * per), b1 = min(it.nseg, b0 + per);
    uint64_t M = 1, A = 0;  // identity
    for (uint32_t s = b0; s < b1; ++s) {
      const uint64_t m = s == 0 ? 0 : (s + 1 == it.nseg ? plast : pseg);
      M = m * M;
      A = m * A + sc.S[it.seg_begin + s];
    }
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {  // lane L holds blocks [L, L + 2*off) after this step
      const uint64_t Mr = __shfl_down_sync(0xffffffffu, M, off);
      const uint64_t Ar = __shfl_down_sync(0xffffffffu, A, off);
      if (lane + off < 32) {
        A = Mr * A + Ar;  // right o left
        M = Mr * M;
      }
    }
    if (lane == 0) *reinterpret_cast<uint64_t*>(it.d.out) = A;
  }
}

int sm_count(int device) {
  static std::mutex mu;
  static std::vector<int> cache;
  std::lock_guard<std::mutex> lk(mu);
  if (size_t(device) >= cache.size()) cache.resize(size_t(device) + 1, 0);
  if (!cache[size_t(device)]) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) n = 148;
    cache[size_t(device)] = n;
  }
  return cache[size_t(device)];
}

template <int K>
void launch_dual(uint32_t grid, uint32_t rgrid, cudaStream_t s, const HashBatch& b, Scratch sc) {
  lzk_fnv_dual_pass_kernel<K><<<grid, kBigThreads, 0, s>>>(b, sc);
  lzk_fnv_resolve_kernel<K><<<rgrid, 256, 0, s>>>(b, sc);
}

void set_pool_threshold(int device) {
  // Keep freed stream-ordered scratch in the device's default pool between
  // calls instead of returning it to the OS at every synchronization.
  static std::mutex mu;
  static std::vector<bool> done;
  std::lock_guard<std::mutex> lk(mu);
  if (size_t(device) >= done.size()) done.resize(size_t(device) + 1, false);
  if (done[size_t(device)]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t keep = 1ull << 30;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  cudaGetLastError();
  done[size_t(device)] = true;
}

int launch_hash(cudaStream_t stream, int device, const lzk_hash_desc* d, uint32_t n, uint32_t max_ctas, bool cont) {
  if (n == 0) return LZK_OK;
  if (d == nullptr) return fail(LZK_ERR_INVALID, "fnv: null descriptor array");
  uint64_t total = 0;
  for (uint32_t i = 0; i < n; ++i) {
    if (d[i].out == 0) return fail(LZK_ERR_INVALID, "fnv: null output address");
    if (d[i].src == 0 && d[i].len) return fail(LZK_ERR_INVALID, "fnv: null source");
    total += d[i].len;
  }
  set_pool_threshold(device);
  const uint32_t ctas = max_ctas ? max_ctas : uint32_t(sm_count(device)) * (kWarpsPerSm / kHashWarps);
  const uint64_t fair = total / (uint64_t(ctas) * kHashWarps);
  // largest first, dealt round-robin to warps (longest-processing-time order)
  std::vector<uint32_t> order(n);
  std::iota(order.begin(), order.end(), 0u);
  std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return d[a].len > d[b].len; });
  std::vector<HashItem> items(n);
  uint32_t segs = 0;
  bool any_long = false;
  for (uint32_t i = 0; i < n; ++i) {
    HashItem& it = items[i];
    it.d = d[order[i]];
    it.seg_begin = segs;
    it.nseg = 1;
    it.seglen = 0;
    const uint64_t body = it.d.len - std::min<uint64_t>(it.d.len, (16u - (it.d.src & 15u)) & 15u);
    if (it.d.len >= kLongMin && it.d.len > 2 * fair) {
      uint64_t sl = std::max<uint64_t>(kSegMin, (body + kMaxSegs - 1) / kMaxSegs);
      sl = (sl + 1023) & ~uint64_t(1023);
      const uint64_t ns = (body + sl - 1) / sl;
      if (ns > 1) {
        it.nseg = uint32_t(ns);
        it.seglen = sl;
        any_long = true;
      }
    }
    segs += it.nseg;
  }
  // stream-ordered device block: item table, then (long ranges) per-segment
  // sums and parities
  const uint64_t table = (uint64_t(n) * sizeof(HashItem) + 255) & ~uint64_t(255);
  const uint64_t bytes = table + (any_long ? uint64_t(segs) * 10 + 16 : 0);
  void* dev = nullptr;
  LZK_CK(cudaMallocAsync(&dev, bytes, stream));
  uint32_t launches = 0;
  thread_local UploadParams up;
  for (uint32_t i = 0; i < n; i += kUploadItems) {
    up.dst = static_cast<HashItem*>(dev) + i;
    up.n = std::min(kUploadItems, n - i);
    up.cont = cont ? 1u : 0u;
    std::copy(items.begin() + i, items.begin() + i + up.n, up.items);
    lzk_fnv_upload_kernel<<<(up.n + 127) / 128, 128, 0, stream>>>(up);
    ++launches;
  }
  HashBatch batch{static_cast<const HashItem*>(dev), n, 0, segs, 0};
  Scratch sc{nullptr, nullptr, nullptr};
  if (any_long) {
    sc.S = reinterpret_cast<uint64_t*>(static_cast<uint8_t*>(dev) + table);
    sc.par = reinterpret_cast<uint8_t*>(sc.S + segs);
    sc.alt = sc.par + segs;
    const cudaError_t me = cudaMemsetAsync(sc.par, 0, 2 * uint64_t(segs), stream);
    if (me != cudaSuccess) {
      cudaFreeAsync(dev, stream);
      return cuda_fail(me, "fnv: scratch memset");
    }
  }
  const uint32_t grid = std::max(1u, std::min<uint32_t>((segs + kHashWarps - 1) / kHashWarps, ctas));
  constexpr uint32_t kSmallPerBig = kBigThreads / kSmallThreads;
  const uint32_t small_warps = kSmallThreads / 32;
  const uint32_t small_grid =
      std::max(1u, std::min<uint32_t>((segs + small_warps - 1) / small_warps, ctas * kSmallPerBig));
  if (any_long) {
    const uint32_t rgrid = (n + 7) / 8;  // resolve: one warp per range
    launch_dual<0>(grid, rgrid, stream, batch, sc);
    launch_dual<1>(grid, rgrid, stream, batch, sc);
    launch_dual<2>(grid, rgrid, stream, batch, sc);
    launch_dual<3>(grid, rgrid, stream, batch, sc);
    launches += 8;
  }
  if (any_long) {
    lzk_fnv_kernel<kBigThreads><<<grid, kBigThreads, 0, stream>>>(batch, sc);
  } else {
    lzk_fnv_kernel<kSmallThreads><<<small_grid, kSmallThreads, 0, stream>>>(batch, sc);
  }
  ++launches;
  if (any_long) {
    lzk_fnv_combine_kernel<<<(n + 7) / 8, 256, 0, stream>>>(batch, sc);
    ++launches;
  }
  cudaError_t e = cudaGetLastError();
  cudaFreeAsync(dev, stream);  // stream-ordered: after the kernels above
  if (e != cudaSuccess) return cuda_fail(e, "lzk_fnv kernels launch");
  lzk_detail::launches.fetch_add(launches, std::memory_order_relaxed);
  return LZK_OK;
}

}  // namespace

extern "C" int lzk_fnv1a64_batch(lzk_stream* s, const lzk_hash_desc* d, uint32_t n, uint32_t max_ctas) {
  if (!s) return fail(LZK_ERR_INVALID, "null stream");
  if (int rc = use_device(s->device)) return rc;
  return launch_hash(s->s, s->device, d, n, max_ctas, false);
}

extern "C" int lzk_fnv1a64_continue(lzk_stream* s, const lzk_hash_desc* d, uint32_t n, uint32_t max_ctas) {
  if (!s) return fail(LZK_ERR_INVALID, "null stream");
  if (int rc = use_device(s->device)) return rc;
  return launch_hash(s->s, s->device, d, n, max_ctas, true);
}
