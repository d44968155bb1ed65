// Internal to liblzk_cuda.so: what the device-layer translation units
// (lzk_cuda.cu: memory, streams, copies; lzk_fnv.cu: checksums) share.
// Nothing here crosses the C ABI.
#ifndef LZK_INTERNAL_H_
#define LZK_INTERNAL_H_

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <string>

#include "lzk_cuda.h"

struct lzk_stream {
  cudaStream_t s = nullptr;
  int device = 0;
  bool owned = true;
};

namespace lzk_detail {

extern thread_local std::string g_err;
extern std::atomic<uint64_t> launches;  // lzk_kernel_launches()

int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);
int use_device(int device);

}  // namespace lzk_detail

#define LZK_CK(call)                                                \
  do {                                                              \
    cudaError_t e_ = (call);                                        \
    if (e_ != cudaSuccess) return lzk_detail::cuda_fail(e_, #call); \
  } while (0)

#endif  // LZK_INTERNAL_H_
