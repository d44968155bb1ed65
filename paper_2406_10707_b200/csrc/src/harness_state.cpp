// See harness_state.hpp.
#include "harness_state.hpp"

#include <algorithm>
#include <cstring>

#include "lzckpt/errors.hpp"
#include "lzckpt/transfer_engine.hpp"
#include "lzk_cuda.h"

namespace lzckpt::detail {

namespace {

void check(int rc, const char* what) {
  if (rc != LZK_OK) throw DeviceError(std::string(what) + ": " + lzk_last_error());
}

std::vector<std::byte> host_bytes(uint64_t n, std::mt19937_64& rng) {
  std::vector<std::byte> out(n);
  for (uint64_t i = 0; i < n; i += 8) {
    const uint64_t w = rng();
    std::memcpy(out.data() + i, &w, std::min<uint64_t>(8, n - i));
  }
  return out;
}

}  // namespace

DeviceState::DeviceState(int device, uint64_t seed) : device_(device), seed_(seed) {
  if (device_ < 0) check(lzk_get_device(&device_), "harness: current device");
  check(lzk_stream_create(device_, 0, &stream_), "harness: stream");
}

DeviceState::~DeviceState() {
  if (stream_) {
    lzk_stream_sync(stream_);
    lzk_stream_destroy(stream_);
  }
}

void DeviceState::fill(size_t index, uint64_t generation, lzk_stream* s) {
  const auto& r = regions_[index];
  // a distinct counter stream per (state, generation, leaf)
  const uint64_t seed = seed_ ^ (0x632BE59BD9B4E019ull * (generation + 1));
  check(lzk_fill_splitmix(s, r->device_ptr(), r->size(), seed, index), "harness: fill");
}

void DeviceState::add(const std::vector<Leaf>& leaves, std::mt19937_64& rng) {
  for (const auto& l : leaves) {
    if (l.region) {
      auto r = std::make_shared<DeviceRegion>(DeviceRegion::Uninitialized{}, l.size, device_);
      regions_.push_back(r);
      fill(regions_.size() - 1, 0, stream_);
      tree_.set_region(l.path, std::move(r));
    } else {
      tree_.set_blob(l.path, host_bytes(l.size, rng));
    }
  }
  sync();
}

void DeviceState::step(uint64_t generation, lzk_stream* on) {
  for (size_t i = 0; i < regions_.size(); ++i) {
    regions_[i]->bump_version();  // declared before the bytes change
    fill(i, generation, on ? on : stream_);
  }
  if (!on) sync();
}

void DeviceState::sync() { check(lzk_stream_sync(stream_), "harness: sync"); }

DeviceState::Image DeviceState::image() const {
  Image img;
  for (const auto& l : tree_.flatten()) {
    img[l.path] = l.region ? std::make_pair(true, l.region->clone_bytes()) : std::make_pair(false, *l.blob);
  }
  return img;
}

std::vector<DeviceState::Leaf> random_layout(const std::string& top, uint64_t bytes, uint64_t large,
                                             uint32_t max_leaves, std::mt19937_64& rng) {
  std::vector<DeviceState::Leaf> out;
  if (bytes == 0) return out;
  const uint64_t head = bytes <= large ? bytes : large + rng() % (bytes - large + 1) / 2;
  std::vector<uint64_t> cuts{head, bytes};
  const uint32_t extra = max_leaves > 2 ? uint32_t(rng() % (max_leaves - 1)) : 0;
  for (uint32_t k = 0; k < extra && bytes > head + 1; ++k) cuts.push_back(head + 1 + rng() % (bytes - head - 1));
  std::sort(cuts.begin(), cuts.end());
  cuts.erase(std::unique(cuts.begin(), cuts.end()), cuts.end());
  static const char* dirs[] = {"blk0", "blk.1", "blk-2", "blk0/sub"};
  uint64_t at = 0;
  for (size_t i = 0; i < cuts.size(); ++i) {
    DeviceState::Leaf l;
    l.size = cuts[i] - at;
    at = cuts[i];
    l.region = i == 0 || rng() % 4 != 0;
    l.path = top + "/" + dirs[i % 4] + "/" + (l.region ? "r" : "b") + std::to_string(i);
    out.push_back(std::move(l));
  }
  return out;
}

}  // namespace lzckpt::detail
