// See numa.hpp. Raw syscalls (mbind, move_pages): libnuma is not required.
#include "numa.hpp"

#include <sched.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <cctype>
#include <cerrno>
#include <filesystem>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

namespace lzckpt::detail {

namespace {

constexpr int kMaxNodes = 1024;
constexpr int kMpolPreferred = 1;
constexpr unsigned kWordBits = 8 * sizeof(unsigned long);

bool node_cpus(int node, cpu_set_t* set) {
  std::ifstream in("/sys/devices/system/node/node" + std::to_string(node) + "/cpulist");
  std::string list;
  if (!in || !std::getline(in, list)) return false;
  CPU_ZERO(set);
  std::stringstream ss(list);
  std::string part;
  bool any = false;
  while (std::getline(ss, part, ',')) {
    if (part.empty()) continue;
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

}  // namespace

int numa_node_count() {
  int n = 0;
  std::error_code ec;
  for (const auto& e : std::filesystem::directory_iterator("/sys/devices/system/node", ec)) {
    const std::string name = e.path().filename().string();
    if (name.rfind("node", 0) == 0 && name.size() > 4 && std::isdigit(static_cast<unsigned char>(name[4]))) ++n;
  }
  return n > 0 ? n : 1;
}

bool bind_thread_to_node(int node) {
  if (node < 0) return false;
  cpu_set_t set;
  if (!node_cpus(node, &set)) return false;
  return sched_setaffinity(0, sizeof set, &set) == 0;
}

bool prefer_node(void* p, uint64_t len, int node) {
  if (node < 0 || node >= kMaxNodes) return false;
  std::vector<unsigned long> mask(kMaxNodes / kWordBits, 0);
  mask[unsigned(node) / kWordBits] = 1ul << (unsigned(node) % kWordBits);
  return syscall(SYS_mbind, p, len, kMpolPreferred, mask.data(), static_cast<unsigned long>(kMaxNodes), 0u) == 0;
}

int page_nodes(const void* p, uint64_t len, uint64_t stride, int* out, uint64_t n) {
  if (stride == 0) stride = 4096;
  std::vector<void*> pages;
  for (uint64_t o = 0; o < len && pages.size() < n; o += stride) {
    pages.push_back(const_cast<char*>(static_cast<const char*>(p) + o));
  }
  std::vector<int> status(pages.size(), 0);
  if (syscall(SYS_move_pages, 0, static_cast<unsigned long>(pages.size()), pages.data(), nullptr, status.data(), 0) !=
      0) {
    return -errno;
  }
  for (size_t i = 0; i < status.size(); ++i) out[i] = status[i];
  return int(status.size());
}

}  // namespace lzckpt::detail
