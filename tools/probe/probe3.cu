// Does the size of the host destination range change CE D2H throughput?
// (100 GB range once vs an 8 GB window reused; THP vs 4K registration.)
#include <cuda_runtime.h>
#include <sys/mman.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <thread>
#include <vector>
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { std::printf("CUDA error %s line %d\n", cudaGetErrorString(e_), __LINE__); std::exit(1);} } while (0)
static char* reg(size_t n, bool thp) {
  char* p = (char*)mmap(nullptr, n, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  if (thp) madvise(p, n, MADV_HUGEPAGE);
  std::vector<std::thread> th;
  for (int t = 0; t < 16; ++t) th.emplace_back([=] { size_t c = n / 16; for (size_t o = c * t; o < c * (t + 1); o += 4096) p[o] = 0; });
  for (auto& t : th) t.join();
  CK(cudaHostRegister(p, n, cudaHostRegisterPortable | cudaHostRegisterMapped));
  return p;
}
int main() {
  system("cat /sys/kernel/mm/transparent_hugepage/enabled /sys/kernel/mm/transparent_hugepage/defrag; grep -i AnonHuge /proc/meminfo; dmesg 2>/dev/null | grep -i -m3 iommu; ls /sys/class/iommu 2>/dev/null");
  CK(cudaSetDevice(0));
  const size_t N = 96ull << 30, W = 8ull << 30, C = 256ull << 20;
  char* d; CK(cudaMalloc(&d, N));
  CK(cudaMemset(d, 3, N));
  cudaStream_t s; CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  for (int thp = 1; thp >= 0; --thp) {
    char* h = reg(N, thp);
    system("grep -i AnonHuge /proc/meminfo");
    auto run = [&](const char* name, auto fn) {
      for (int r = 0; r < 2; ++r) {
        CK(cudaEventRecord(a, s)); fn(); CK(cudaEventRecord(b, s)); CK(cudaEventSynchronize(b));
        float ms; CK(cudaEventElapsedTime(&ms, a, b));
        std::printf("%s %-44s %6.2f GB/s\n", thp ? "THP" : "4K ", name, N / (ms * 1e-3) / 1e9);
      }
    };
    run("96 GB range, 256 MB chunks", [&] { for (size_t o = 0; o < N; o += C) CK(cudaMemcpyAsync(h + o, d + o, C, cudaMemcpyDeviceToHost, s)); });
    run("8 GB window x12, 256 MB chunks", [&] { for (size_t o = 0; o < N; o += C) CK(cudaMemcpyAsync(h + (o % W), d + o, C, cudaMemcpyDeviceToHost, s)); });
    run("96 GB range, 64 MB chunks", [&] { for (size_t o = 0; o < N; o += C / 4) CK(cudaMemcpyAsync(h + o, d + o, C / 4, cudaMemcpyDeviceToHost, s)); });
    run("src 8 GB window x12 -> 96 GB dst", [&] { for (size_t o = 0; o < N; o += C) CK(cudaMemcpyAsync(h + o, d + (o % W), C, cudaMemcpyDeviceToHost, s)); });
    CK(cudaHostUnregister(h));
    munmap(h, N);
  }
  return 0;
}
