// Cross-process uplink relay probe (two processes, two GPUs).
//
// The owner process (GPU A) holds the source bytes in HBM and its pinned ring
// in a memfd-backed shared mapping. The helper process (GPU B) maps the same
// ring (open /proc/<owner>/fd/<memfd>, mmap, cudaHostRegister), opens the
// owner's buffer through CUDA IPC, and runs a copy kernel on ITS OWN GPU that
// reads A's HBM over NVLink and stores into the ring over B's PCIe link,
// while the owner's copy engine moves the other part over A's link.
// Checks the bytes and reports aggregate GB/s and the pinning costs.
//
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o relay_ipc_probe relay_ipc_probe.cu
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/wait.h>
#include <unistd.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#define CK(x)                                                                                 \
  do {                                                                                        \
    cudaError_t e_ = (x);                                                                     \
    if (e_ != cudaSuccess) {                                                                  \
      std::fprintf(stderr, "[%d] %s:%d %s: %s\n", getpid(), __FILE__, __LINE__, #x,          \
                   cudaGetErrorString(e_));                                                   \
      std::exit(1);                                                                           \
    }                                                                                         \
  } while (0)

__global__ void copy_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n16) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n16; i += size_t(gridDim.x) * blockDim.x) {
    dst[i] = src[i];
  }
}

__global__ void fill_kernel(uint64_t* p, size_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    p[i] = i * 0x9E3779B97F4A7C15ull + 12345;
  }
}

double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

struct Msg {
  int owner_pid;
  int memfd;
  cudaIpcMemHandle_t mem;
  cudaIpcEventHandle_t start;  // recorded by the owner when the source is ready
};

void write_all(int fd, const void* p, size_t n) {
  const char* c = static_cast<const char*>(p);
  while (n) {
    ssize_t w = write(fd, c, n);
    if (w <= 0) std::exit(2);
    c += w;
    n -= size_t(w);
  }
}
void read_all(int fd, void* p, size_t n) {
  char* c = static_cast<char*>(p);
  while (n) {
    ssize_t r = read(fd, c, n);
    if (r <= 0) std::exit(3);
    c += r;
    n -= size_t(r);
  }
}

int main(int argc, char** argv) {
  const int A = argc > 1 ? std::atoi(argv[1]) : 0;
  const int B = argc > 2 ? std::atoi(argv[2]) : 1;
  const double share = argc > 3 ? std::atof(argv[3]) : 0.5;  // fraction relayed through B
  const bool priv = argc > 4 && std::string(argv[4]) == "private";
  const size_t bytes = 8ull << 30;
  const size_t split = (size_t(double(bytes) * (1.0 - share)) / 4096) * 4096;
  int to_helper[2], to_owner[2];
  if (pipe(to_helper) || pipe(to_owner)) return 4;

  // ring: memfd shared mapping, created before fork so both can reach it
  const int memfd = memfd_create("lzk_ring", 0);
  if (memfd < 0 || ftruncate(memfd, off_t(bytes))) return 5;

  const pid_t child = fork();
  if (child == 0) {  // ---------------- helper (GPU B)
    Msg m;
    read_all(to_helper[0], &m, sizeof m);
    void* ring = nullptr;
    double t0 = now();
    if (priv) {  // the helper's own pinned staging (it would write the owner's file itself)
      CK(cudaSetDevice(B));
      CK(cudaHostAlloc(&ring, bytes, cudaHostAllocPortable | cudaHostAllocMapped));
      std::printf("helper: private pinned staging %zu GiB: %.2f s\n", bytes >> 30, now() - t0);
    } else {
      const std::string path = "/proc/" + std::to_string(m.owner_pid) + "/fd/" + std::to_string(m.memfd);
      const int fd = open(path.c_str(), O_RDWR);
      if (fd < 0) {
        std::perror("open memfd");
        return 6;
      }
      ring = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
      if (ring == MAP_FAILED) return 7;
      CK(cudaSetDevice(B));
      CK(cudaHostRegister(ring, bytes, cudaHostRegisterPortable | cudaHostRegisterMapped));
      std::printf("helper: cudaHostRegister of the owner's %zu GiB ring: %.2f s\n", bytes >> 30, now() - t0);
    }
    int can = 0;
    CK(cudaDeviceCanAccessPeer(&can, B, A));
    if (can) CK(cudaDeviceEnablePeerAccess(A, 0));
    void* src = nullptr;
    t0 = now();
    CK(cudaIpcOpenMemHandle(&src, m.mem, cudaIpcMemLazyEnablePeerAccess));
    std::printf("helper: IPC open %.3f ms (peer %d)\n", (now() - t0) * 1e3, can);
    cudaEvent_t start;
    CK(cudaIpcOpenEventHandle(&start, m.start));
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    for (int rep = 0; rep < 5; ++rep) {
      char go;
      read_all(to_helper[0], &go, 1);
      CK(cudaStreamWaitEvent(s, start, 0));  // producer ordering across processes
      const double h0 = now();
      copy_kernel<<<16, 512, 0, s>>>(reinterpret_cast<const uint4*>(static_cast<char*>(src) + split),
                                     reinterpret_cast<uint4*>(static_cast<char*>(ring) + split), (bytes - split) / 16);
      CK(cudaGetLastError());
      CK(cudaStreamSynchronize(s));
      const double dt = now() - h0;
      write_all(to_owner[1], &dt, sizeof dt);
    }
    // check the relayed part
    size_t bad = 0;
    const uint64_t* r = static_cast<const uint64_t*>(ring);
    for (size_t i = split / 8; i < bytes / 8; i += 511) bad += r[i] != i * 0x9E3779B97F4A7C15ull + 12345;
    std::printf("helper: relayed part mismatches %zu\n", bad);
    CK(cudaIpcCloseMemHandle(src));
    if (priv) {
      CK(cudaFreeHost(ring));
    } else {
      CK(cudaHostUnregister(ring));
    }
    return 0;
  }

  // ---------------- owner (GPU A)
  CK(cudaSetDevice(A));
  void* ring = nullptr;
  double t0 = now();
  if (priv) {
    CK(cudaHostAlloc(&ring, bytes, cudaHostAllocPortable | cudaHostAllocMapped));
    std::printf("owner: private pinned ring %zu GiB: %.2f s\n", bytes >> 30, now() - t0);
  } else {
  ring = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_SHARED, memfd, 0);
  if (ring == MAP_FAILED) return 8;
  {
    std::vector<std::thread> th;
    for (int t = 0; t < 16; ++t) {
      th.emplace_back([&, t] {
        for (size_t o = size_t(t) * 4096; o < bytes; o += 16 * 4096) static_cast<volatile char*>(ring)[o] = 0;
      });
    }
    for (auto& x : th) x.join();
  }
  const double t_touch = now() - t0;
  t0 = now();
  CK(cudaHostRegister(ring, bytes, cudaHostRegisterPortable | cudaHostRegisterMapped));
  std::printf("owner: memfd ring %zu GiB: first touch %.2f s, cudaHostRegister %.2f s (4 KiB shmem pages)\n",
              bytes >> 30, t_touch, now() - t0);
  }
  void* src = nullptr;
  CK(cudaMalloc(&src, bytes));
  fill_kernel<<<1024, 256>>>(static_cast<uint64_t*>(src), bytes / 8);
  CK(cudaDeviceSynchronize());
  cudaEvent_t start;
  CK(cudaEventCreateWithFlags(&start, cudaEventDisableTiming | cudaEventInterprocess));
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  CK(cudaEventRecord(start, s));
  Msg m;
  m.owner_pid = getpid();
  m.memfd = memfd;
  CK(cudaIpcGetMemHandle(&m.mem, src));
  CK(cudaIpcGetEventHandle(&m.start, start));
  write_all(to_helper[1], &m, sizeof m);

  double best = 0, best_own = 0, best_helper = 0;
  for (int rep = 0; rep < 5; ++rep) {
    std::memset(ring, 0, 4096);
    CK(cudaEventRecord(start, s));
    const double h0 = now();
    char go = 1;
    write_all(to_helper[1], &go, 1);
    for (size_t o = 0; o < split; o += 256ull << 20) {
      CK(cudaMemcpyAsync(static_cast<char*>(ring) + o, static_cast<char*>(src) + o,
                         std::min<size_t>(256ull << 20, split - o), cudaMemcpyDeviceToHost, s));
    }
    CK(cudaStreamSynchronize(s));
    const double own = now() - h0;
    double helper = 0;
    read_all(to_owner[0], &helper, sizeof helper);
    const double all = now() - h0;
    best = std::max(best, bytes / all / 1e9);
    best_own = std::max(best_own, split / own / 1e9);
    best_helper = std::max(best_helper, (bytes - split) / helper / 1e9);
  }
  // verify every 4 KiB word 0.. in both parts
  size_t bad = 0;
  const uint64_t* r = static_cast<const uint64_t*>(ring);
  for (size_t i = 0; i < (priv ? split : bytes) / 8; i += 511) bad += r[i] != i * 0x9E3779B97F4A7C15ull + 12345;
  std::printf("owner: share %.2f relayed via GPU %d: aggregate %.2f GB/s (own link %.2f, relay %.2f); mismatches %zu\n",
              share, B, best, best_own, best_helper, bad);
  int st = 0;
  waitpid(child, &st, 0);
  return bad ? 9 : 0;
}
