// NUMA placement for one rank's host-side resources (the
// pinned pool lives on the GPU's NUMA node, and so do the threads that touch
// it). The reference pool is a plain std::vector (buffer_pool.cpp:10) and its
// copy/flush workers float; on a two-socket 8-GPU host that sends every
// snapshot byte across the socket interconnect. No-ops on single-node hosts.
#pragma once

#include <cstdint>

namespace lzckpt::detail {

// Number of NUMA nodes the kernel reports (1 on single-node machines).
int numa_node_count();
// Pins the calling thread to the CPUs of `node`; returns false (and leaves
// the affinity alone) for node < 0 or an unreadable cpulist.
bool bind_thread_to_node(int node);
// MPOL_PREFERRED on `node` for [p, p+len), to be set before the first touch.
bool prefer_node(void* p, uint64_t len, int node);
// Node currently holding each page (move_pages(2) query); -errno per page
// that is not resident.
int page_nodes(const void* p, uint64_t len, uint64_t stride, int* out, uint64_t n);

}  // namespace lzckpt::detail
