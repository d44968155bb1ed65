// Synthetic rank state for the verify and bench harnesses, resident in HBM.
//
// The reference harnesses keep "device" state in host vectors and mutate it
// with memcpy (verify.cpp, bench.cpp). Here the state is what a trainer has:
// real device allocations written by kernels. Regions are filled and every
// "optimizer step" rewrites them ON the device (splitmix64 fill kernel, a new
// stream per generation), declaring the mutation with a version bump first so
// torn detection sees it exactly as it sees DeviceRegion::mutate. Images for
// the byte-exact checks are read back from the device.
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <random>
#include <string>
#include <utility>
#include <vector>

#include "lzckpt/state_tree.hpp"

struct lzk_stream;

namespace lzckpt::detail {

class DeviceState {
 public:
  // One leaf of a shard layout.
  struct Leaf {
    std::string path;
    uint64_t size = 0;
    bool region = true;
  };
  // path -> (is_region, bytes)
  using Image = std::map<std::string, std::pair<bool, std::vector<std::byte>>>;

  DeviceState(int device, uint64_t seed);
  ~DeviceState();
  DeviceState(const DeviceState&) = delete;
  DeviceState& operator=(const DeviceState&) = delete;

  // Materialises leaves: regions in HBM, filled on the device with
  // generation 0; blobs as host bytes from `rng`.
  void add(const std::vector<Leaf>& leaves, std::mt19937_64& rng);
  // The optimizer step: every region is declared mutated, then rewritten on
  // the device with `generation`'s stream — on `on` (e.g. the trainer's
  // compute stream, behind its lazy fence) without waiting, or on the
  // state's own stream, waited for.
  void step(uint64_t generation, lzk_stream* on = nullptr);
  void sync();
  Image image() const;

  StateTree& tree() { return tree_; }
  const StateTree& tree() const { return tree_; }
  int device() const { return device_; }

 private:
  void fill(size_t index, uint64_t generation, lzk_stream* s);

  int device_;
  uint64_t seed_;
  lzk_stream* stream_ = nullptr;
  StateTree tree_;
  std::vector<std::shared_ptr<DeviceRegion>> regions_;  // fill order = leaf index
};

// Splits `bytes` into a random leaf mix under `top`: the first leaf is a
// region of at least `large` bytes (a streamed entry), then up to `max_leaves`
// pieces cut at random points, each a region or (1 in 4) a host blob, paths
// spread over a few subdirectories to exercise per-component ordering.
std::vector<DeviceState::Leaf> random_layout(const std::string& top, uint64_t bytes, uint64_t large,
                                             uint32_t max_leaves, std::mt19937_64& rng);

}  // namespace lzckpt::detail
