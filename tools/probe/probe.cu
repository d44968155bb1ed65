// Hardware probe for the snapshot path: host-link D2H rates of the copy engine
// and of SM stores into mapped pinned memory. Throwaway measurement tool.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <chrono>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); std::exit(1);} } while (0)

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

// each CTA copies a contiguous block of the range (better locality of host writes)
__global__ void store_kernel_blocked(const uint4* __restrict__ src, uint4* dst, size_t n16, size_t per_cta) {
  size_t b = (size_t)blockIdx.x * per_cta;
  size_t e = b + per_cta; if (e > n16) e = n16;
  for (size_t i = b + threadIdx.x; i < e; i += blockDim.x * 4) {
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) { size_t j = i + u * blockDim.x; if (j < e) v[u] = src[j]; }
#pragma unroll
    for (int u = 0; u < 4; ++u) { size_t j = i + u * blockDim.x; if (j < e) dst[j] = v[u]; }
  }
}

int main() {
  int dev = 0; CK(cudaSetDevice(dev));
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  std::printf("device %s SMs %d pciBus %d\n", p.name, p.multiProcessorCount, p.pciBusID);
  const size_t N = 4ull << 30;
  void* d; CK(cudaMalloc(&d, N + 4096));
  CK(cudaMemset(d, 1, N));
  auto t0 = std::chrono::steady_clock::now();
  void* h; CK(cudaHostAlloc(&h, N + 4096, cudaHostAllocMapped | cudaHostAllocPortable));
  auto t1 = std::chrono::steady_clock::now();
  std::printf("cudaHostAlloc %zu GiB: %.3f s\n", N >> 30, std::chrono::duration<double>(t1 - t0).count());
  void* hd; CK(cudaHostGetDevicePointer(&hd, h, 0));
  std::printf("mapped alias same as host ptr: %d\n", hd == h);
  cudaStream_t s; CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  auto tm = [&](auto fn, size_t bytes, const char* name) {
    for (int w = 0; w < 2; ++w) fn();
    CK(cudaStreamSynchronize(s));
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
      CK(cudaEventRecord(a, s)); fn(); CK(cudaEventRecord(b, s)); CK(cudaEventSynchronize(b));
      float ms; CK(cudaEventElapsedTime(&ms, a, b)); if (ms < best) best = ms;
    }
    std::printf("%-48s %8.2f GB/s (%.3f ms)\n", name, bytes / (best * 1e-3) / 1e9, best);
  };
  tm([&] { CK(cudaMemcpyAsync(h, d, N, cudaMemcpyDeviceToHost, s)); }, N, "CE D2H 4GiB aligned");
  tm([&] { CK(cudaMemcpyAsync((char*)h + 14, d, N, cudaMemcpyDeviceToHost, s)); }, N, "CE D2H 4GiB dst+14");
  tm([&] { CK(cudaMemcpyAsync((char*)h + 14, (char*)d + 3, N, cudaMemcpyDeviceToHost, s)); }, N, "CE D2H 4GiB dst+14 src+3");
  tm([&] { CK(cudaMemcpyAsync(d, h, N, cudaMemcpyHostToDevice, s)); }, N, "CE H2D 4GiB");
  for (size_t sz : {4096ul, 65536ul, 1ul << 20, 16ul << 20}) {
    size_t cnt = std::min<size_t>(N / sz, 20000);
    char name[96]; std::snprintf(name, sizeof name, "CE D2H %zu x %zu B", cnt, sz);
    tm([&] { for (size_t i = 0; i < cnt; ++i) CK(cudaMemcpyAsync((char*)h + i * sz, (char*)d + i * sz, sz, cudaMemcpyDeviceToHost, s)); }, cnt * sz, name);
  }
  size_t n16 = N / 16;
  for (int threads : {256, 512, 1024}) {
    for (int ctas : {1, 2, 4, 8, 16, 32, 64, 148, 296}) {
      char name[96]; std::snprintf(name, sizeof name, "SM store gridstride %d x %d", ctas, threads);
      tm([&] { store_kernel<<<ctas, threads, 0, s>>>((const uint4*)d, (uint4*)hd, n16); }, N, name);
      std::snprintf(name, sizeof name, "SM store blocked %d x %d", ctas, threads);
      size_t per = (n16 + ctas - 1) / ctas;
      tm([&] { store_kernel_blocked<<<ctas, threads, 0, s>>>((const uint4*)d, (uint4*)hd, n16, per); }, N, name);
    }
  }
  // concurrent CE + SM stores (is the link the limit?)
  cudaStream_t s2; CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  {
    auto fn = [&] {
      CK(cudaMemcpyAsync(h, d, N / 2, cudaMemcpyDeviceToHost, s));
      store_kernel<<<16, 512, 0, s2>>>((const uint4*)((char*)d + N / 2), (uint4*)((char*)hd + N / 2), n16 / 2);
    };
    fn(); CK(cudaDeviceSynchronize());
    auto c0 = std::chrono::steady_clock::now();
    fn(); CK(cudaDeviceSynchronize());
    auto c1 = std::chrono::steady_clock::now();
    std::printf("CE+SM concurrent 2x2GiB: %.2f GB/s\n", N / std::chrono::duration<double>(c1 - c0).count() / 1e9);
  }
  return 0;
}
