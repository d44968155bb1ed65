// Synthetic shard workloads for tests and bench.
// Reads the spec text written by paper_2406_10707_b200/workloads.py and
// materializes the state tree in HBM: splitmix64 leaves are generated on the
// GPU (lzk_fill_splitmix), mt19937_64 leaves on the host (the generator is
// sequential) and uploaded.
#pragma once

#include <cstdint>
#include <string>

#include "lzckpt/state_tree.hpp"
#include "lzckpt/topology.hpp"

namespace lzckpt {

struct Workload {
  StateTree tree;
  ModelSpec model;
  ParallelTopology topo;
  RankCoord rank;
  uint64_t step = 1;
  uint64_t leaves = 0;
  uint64_t bytes = 0;
};

Workload build_workload(const std::string& spec_path, int device);

}  // namespace lzckpt
