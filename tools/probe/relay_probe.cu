// Uplink-relay probe (one process, two GPUs): can GPU B carry GPU A's
// snapshot bytes to host memory over B's own PCIe link, reading A's HBM over
// NVLink? Measures, with CUDA events, 8 GiB device->pinned host:
//   a   A's copy engine, A's memory -> host
//   b   B's copy engine, A's memory (peer) -> host
//   ab  a and b at once on disjoint halves (aggregate)
//   k   a gather-style SM kernel on B reading A's memory, storing to host
//   ak  a (copy engine on A) and k at once
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o relay_probe relay_probe.cu
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                                     \
  do {                                                                                            \
    cudaError_t e_ = (x);                                                                         \
    if (e_ != cudaSuccess) {                                                                      \
      std::fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_));     \
      std::exit(1);                                                                               \
    }                                                                                             \
  } while (0)

__global__ void copy_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n16) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n16; i += size_t(gridDim.x) * blockDim.x) {
    dst[i] = src[i];
  }
}

double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

int main(int argc, char** argv) {
  const int A = argc > 1 ? std::atoi(argv[1]) : 0;
  const int B = argc > 2 ? std::atoi(argv[2]) : 1;
  const size_t bytes = 8ull << 30, chunk = 256ull << 20;
  int can = 0;
  CK(cudaDeviceCanAccessPeer(&can, B, A));
  std::printf("peer access %d -> %d: %d\n", B, A, can);
  void* src = nullptr;
  CK(cudaSetDevice(A));
  CK(cudaMalloc(&src, bytes));
  CK(cudaMemset(src, 0x5a, bytes));
  void* host = nullptr;
  CK(cudaHostAlloc(&host, bytes, cudaHostAllocPortable | cudaHostAllocMapped));
  CK(cudaSetDevice(B));
  if (can) CK(cudaDeviceEnablePeerAccess(A, 0));
  cudaStream_t sa, sb;
  CK(cudaSetDevice(A));
  CK(cudaStreamCreateWithFlags(&sa, cudaStreamNonBlocking));
  CK(cudaSetDevice(B));
  CK(cudaStreamCreateWithFlags(&sb, cudaStreamNonBlocking));

  auto ce = [&](cudaStream_t s, int dev, size_t off, size_t len) {
    CK(cudaSetDevice(dev));
    for (size_t o = 0; o < len; o += chunk) {
      CK(cudaMemcpyAsync(static_cast<char*>(host) + off + o, static_cast<char*>(src) + off + o,
                         std::min(chunk, len - o), cudaMemcpyDefault, s));
    }
  };
  auto kern = [&](size_t off, size_t len) {
    CK(cudaSetDevice(B));
    copy_kernel<<<16, 512, 0, sb>>>(reinterpret_cast<const uint4*>(static_cast<char*>(src) + off),
                                    reinterpret_cast<uint4*>(static_cast<char*>(host) + off), len / 16);
    CK(cudaGetLastError());
  };
  auto sync = [&] {
    CK(cudaStreamSynchronize(sa));
    CK(cudaStreamSynchronize(sb));
  };
  // per-stream elapsed time (events on A's and B's streams around fn)
  cudaEvent_t a0, a1, b0, b1;
  CK(cudaSetDevice(A));
  CK(cudaEventCreate(&a0));
  CK(cudaEventCreate(&a1));
  CK(cudaSetDevice(B));
  CK(cudaEventCreate(&b0));
  CK(cudaEventCreate(&b1));
  auto run = [&](const char* name, auto fn, size_t moved) {
    fn();
    sync();  // warm-up
    double best = 0;
    float ta = 0, tb = 0;
    for (int r = 0; r < 4; ++r) {
      CK(cudaSetDevice(A));
      CK(cudaEventRecord(a0, sa));
      CK(cudaSetDevice(B));
      CK(cudaEventRecord(b0, sb));
      const double t0 = now();
      fn();
      CK(cudaSetDevice(A));
      CK(cudaEventRecord(a1, sa));
      CK(cudaSetDevice(B));
      CK(cudaEventRecord(b1, sb));
      sync();
      const double gbps = moved / (now() - t0) / 1e9;
      if (gbps > best) {
        best = gbps;
        CK(cudaEventElapsedTime(&ta, a0, a1));
        CK(cudaEventElapsedTime(&tb, b0, b1));
      }
    }
    std::printf("%-8s %8.2f GB/s   (A stream %.1f ms, B stream %.1f ms)\n", name, best, ta, tb);
  };
  run("a", [&] { ce(sa, A, 0, bytes); }, bytes);
  run("b", [&] { ce(sb, B, 0, bytes); }, bytes);
  run("ab", [&] { ce(sa, A, 0, bytes / 2); ce(sb, B, bytes / 2, bytes / 2); }, bytes);
  run("ab31", [&] { ce(sa, A, 0, bytes / 4 * 3); ce(sb, B, bytes / 4 * 3, bytes / 4); }, bytes);
  if (can) {
    run("k", [&] { kern(0, bytes); }, bytes);
    run("ak", [&] { ce(sa, A, 0, bytes / 2); kern(bytes / 2, bytes / 2); }, bytes);
    // copy engines only: A's memory -> B's HBM over NVLink (D2D), then B's
    // HBM -> host over B's link, two chunks in flight on two streams
    CK(cudaSetDevice(B));
    void* stage = nullptr;
    CK(cudaMalloc(&stage, 2 * chunk));  // two slots of the largest chunk size
    cudaStream_t sb2;
    CK(cudaStreamCreateWithFlags(&sb2, cudaStreamNonBlocking));
    cudaEvent_t in_done[2], out_done[2];
    for (int k = 0; k < 2; ++k) {
      CK(cudaEventCreateWithFlags(&in_done[k], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&out_done[k], cudaEventDisableTiming));
      CK(cudaEventRecord(out_done[k], sb));
    }
    auto dd = [&](size_t off, size_t len, size_t step = 0) {
      if (step == 0) step = chunk;
      CK(cudaSetDevice(B));
      int k = 0;
      for (size_t o = 0; o < len; o += step, k ^= 1) {
        const size_t n = std::min(step, len - o);
        char* st = static_cast<char*>(stage) + k * chunk;
        CK(cudaStreamWaitEvent(sb2, out_done[k], 0));
        CK(cudaMemcpyAsync(st, static_cast<char*>(src) + off + o, n, cudaMemcpyDefault, sb2));
        CK(cudaEventRecord(in_done[k], sb2));
        CK(cudaStreamWaitEvent(sb, in_done[k], 0));
        CK(cudaMemcpyAsync(static_cast<char*>(host) + off + o, st, n, cudaMemcpyDeviceToHost, sb));
        CK(cudaEventRecord(out_done[k], sb));
      }
    };
    run("dd", [&] { dd(0, bytes); }, bytes);
    run("add", [&] { ce(sa, A, 0, bytes / 2); dd(bytes / 2, bytes / 2); }, bytes);
    // the same with smaller pull/push chunks: the NVLink pull of A's memory
    // runs in shorter bursts (does A's own DMA lose less?)
    for (size_t mib : {64, 16, 4}) {
      char name[16];
      std::snprintf(name, sizeof name, "add%zu", mib);
      run(name, [&] { ce(sa, A, 0, bytes / 2); dd(bytes / 2, bytes / 2, mib << 20); }, bytes);
    }
    // the pull alone (A's memory -> B's HBM): ~NVLink rate, or a PCIe rate
    // when the peer path is not NVLink
    run("pull", [&] {
      CK(cudaSetDevice(B));
      for (size_t o = 0; o < bytes; o += chunk) {
        CK(cudaMemcpyAsync(stage, static_cast<char*>(src) + o, chunk, cudaMemcpyDefault, sb));
      }
    }, bytes);
    // A's own DMA alone over the same half, for the split
    run("a_half", [&] { ce(sa, A, 0, bytes / 2); }, bytes / 2);
    run("dd_half", [&] { dd(bytes / 2, bytes / 2); }, bytes / 2);
    CK(cudaStreamSynchronize(sb2));
  }
  return 0;
}
