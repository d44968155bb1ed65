// Host-link experiments for the snapshot path: does the pinned-memory flavour
// (cudaHostAlloc vs mmap+THP+cudaHostRegister vs 4K pages+register), the DMA
// chunk size, per-chunk events, or a TMA bulk store change D2H throughput?
#include <cuda_runtime.h>
#include <sys/mman.h>

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); std::exit(1);} } while (0)

static void* host_mem(size_t n, int kind) {
  if (kind == 0) {
    void* p; CK(cudaHostAlloc(&p, n, cudaHostAllocMapped | cudaHostAllocPortable)); return p;
  }
  void* p = mmap(nullptr, n, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  if (kind == 1) madvise(p, n, MADV_HUGEPAGE);
  std::vector<std::thread> th;
  for (int t = 0; t < 16; ++t) th.emplace_back([=] { size_t c = n / 16; for (size_t o = c * t; o < c * (t + 1); o += 4096) ((volatile char*)p)[o] = 0; });
  for (auto& t : th) t.join();
  CK(cudaHostRegister(p, n, cudaHostRegisterPortable | cudaHostRegisterMapped));
  return p;
}

__global__ void store_kernel(const uint4* __restrict__ src, uint4* dst, size_t n16) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride * 4) {
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) { size_t j = i + u * stride; if (j < n16) v[u] = src[j]; }
#pragma unroll
    for (int u = 0; u < 4; ++u) { size_t j = i + u * stride; if (j < n16) dst[j] = v[u]; }
  }
}

// TMA bulk store: stage CHUNK bytes in smem, one thread issues
// cp.async.bulk.global.shared::cta to the (host-mapped) destination.
template <int CHUNK>
__global__ void bulk_store_kernel(const uint4* __restrict__ src, char* dst, size_t n) {
  extern __shared__ __align__(128) uint4 smem[];
  const size_t nchunks = n / CHUNK;
  for (size_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const uint4* s = src + c * (CHUNK / 16);
    for (int i = threadIdx.x; i < CHUNK / 16; i += blockDim.x) smem[i] = s[i];
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + c * CHUNK), "r"(sa), "r"(CHUNK) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  CK(cudaSetDevice(0));
  const size_t N = 8ull << 30;
  void* d; CK(cudaMalloc(&d, N));
  CK(cudaMemset(d, 7, N));
  cudaStream_t s; CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  std::vector<cudaEvent_t> evs(4096);
  for (auto& ev : evs) CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  const char* kinds[] = {"cudaHostAlloc", "mmap+THP+register", "mmap4K+register"};
  for (int kind = 0; kind < 3; ++kind) {
    auto t0 = std::chrono::steady_clock::now();
    char* h = (char*)host_mem(N, kind);
    double pin_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::printf("== %s (pin %.2f s for 8 GiB)\n", kinds[kind], pin_s);
    auto run = [&](const char* name, auto fn) {
      fn(); CK(cudaStreamSynchronize(s));
      float best = 1e30f, tot = 0;
      for (int r = 0; r < 3; ++r) {
        CK(cudaEventRecord(a, s)); fn(); CK(cudaEventRecord(b, s)); CK(cudaEventSynchronize(b));
        float ms; CK(cudaEventElapsedTime(&ms, a, b)); best = ms < best ? ms : best; tot += ms;
      }
      std::printf("  %-40s best %6.2f GB/s  mean %6.2f GB/s\n", name, N / (best * 1e-3) / 1e9, 3 * N / (tot * 1e-3) / 1e9);
    };
    for (size_t chunk : {4ul << 20, 16ul << 20, 64ul << 20, 256ul << 20, 1ul << 30}) {
      char name[64]; std::snprintf(name, sizeof name, "CE chunk %zu MiB", chunk >> 20);
      run(name, [&] { for (size_t o = 0; o < N; o += chunk) CK(cudaMemcpyAsync(h + o, (char*)d + o, chunk, cudaMemcpyDeviceToHost, s)); });
      std::snprintf(name, sizeof name, "CE chunk %zu MiB + event each", chunk >> 20);
      run(name, [&] { size_t k = 0; for (size_t o = 0; o < N; o += chunk) { CK(cudaMemcpyAsync(h + o, (char*)d + o, chunk, cudaMemcpyDeviceToHost, s)); CK(cudaEventRecord(evs[k++ % evs.size()], s)); } });
    }
    run("CE chunk 64 MiB dst+6", [&] { for (size_t o = 0; o + (64ul << 20) < N; o += 64ul << 20) CK(cudaMemcpyAsync(h + o + 6, (char*)d + o, 64ul << 20, cudaMemcpyDeviceToHost, s)); });
    for (int ctas : {8, 16, 32}) {
      char name[64]; std::snprintf(name, sizeof name, "SM store %d x 512", ctas);
      run(name, [&] { store_kernel<<<ctas, 512, 0, s>>>((const uint4*)d, (uint4*)h, N / 16); });
    }
    CK(cudaFuncSetAttribute(bulk_store_kernel<32768>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768));
    for (int ctas : {8, 16, 32, 64}) {
      char name[64]; std::snprintf(name, sizeof name, "TMA bulk store 32K x %d CTAs", ctas);
      run(name, [&] { bulk_store_kernel<32768><<<ctas, 256, 32768, s>>>((const uint4*)d, h, N); });
      CK(cudaGetLastError());
    }
    // correctness of the bulk store
    CK(cudaMemset(d, 0x5a, 1 << 20)); memset(h, 0, 1 << 20);
    bulk_store_kernel<32768><<<8, 256, 32768, s>>>((const uint4*)d, h, 1 << 20); CK(cudaStreamSynchronize(s));
    int bad = 0; for (int i = 0; i < (1 << 20); ++i) bad += (unsigned char)h[i] != 0x5a;
    std::printf("  bulk store check: %d bad bytes\n", bad);
    if (kind == 0) CK(cudaFreeHost(h)); else { CK(cudaHostUnregister(h)); munmap(h, N); }
  }
  return 0;
}
