// Spec reader + device materialization; see include/lzckpt/workload.hpp.
#include "lzckpt/workload.hpp"

#include <cstring>
#include <fstream>
#include <random>
#include <sstream>

#include "lzckpt/errors.hpp"
#include "lzk_cuda.h"

namespace lzckpt {

namespace {

uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

void fill_splitmix_host(std::vector<std::byte>& b, uint64_t seed, uint64_t leaf) {
  const uint64_t base = seed ^ (leaf * 0xD1B54A32D192ED03ull);
  uint64_t w = 0, k = 0;
  for (; k + 8 <= b.size(); k += 8, ++w) {
    const uint64_t v = mix64(base + (w + 1) * 0x9E3779B97F4A7C15ull);
    std::memcpy(b.data() + k, &v, 8);
  }
  if (k < b.size()) {
    const uint64_t v = mix64(base + (w + 1) * 0x9E3779B97F4A7C15ull);
    std::memcpy(b.data() + k, &v, b.size() - k);
  }
}

void fill_mt(std::vector<std::byte>& b, std::mt19937_64& rng) {
  uint64_t k = 0;
  for (; k + 8 <= b.size(); k += 8) {
    const uint64_t w = rng();
    std::memcpy(b.data() + k, &w, 8);
  }
  if (k < b.size()) {
    const uint64_t w = rng();
    std::memcpy(b.data() + k, &w, b.size() - k);
  }
}

}  // namespace

Workload build_workload(const std::string& spec_path, int device) {
  std::ifstream in(spec_path);
  if (!in) throw IoError("cannot open workload spec " + spec_path);
  Workload w;
  std::string gen = "splitmix64";
  uint64_t seed = 0;
  struct Leaf {
    bool region;
    std::string path;
    uint64_t size;
  };
  std::vector<Leaf> leaves;
  std::string line;
  while (std::getline(in, line)) {
    if (line.empty() || line[0] == '#') continue;
    std::istringstream ls(line);
    std::string kw;
    ls >> kw;
    if (kw == "model") {
      ls >> w.model.param_count >> w.model.layer_count >> w.model.bytes_per_param_model >>
          w.model.bytes_per_param_optimizer;
    } else if (kw == "topology") {
      ls >> w.topo.dp >> w.topo.pp >> w.topo.tp >> w.topo.gpus_per_node >> w.topo.node_count;
    } else if (kw == "rank") {
      ls >> w.rank.dp >> w.rank.pp >> w.rank.tp;
    } else if (kw == "step") {
      ls >> w.step;
    } else if (kw == "gen") {
      ls >> gen >> seed;
    } else if (kw == "leaf") {
      Leaf l;
      std::string kind;
      ls >> kind >> l.path >> l.size;
      l.region = kind == "r";
      leaves.push_back(std::move(l));
    } else {
      throw ConfigError("workload spec: unknown directive '" + kw + "'");
    }
  }
  if (gen != "splitmix64" && gen != "mt19937_64") throw ConfigError("workload spec: unknown generator " + gen);

  lzk_stream* s = nullptr;
  if (lzk_stream_create(device, 0, &s) != LZK_OK) throw DeviceError(std::string("workload stream: ") + lzk_last_error());
  struct Guard {
    lzk_stream* s;
    ~Guard() { lzk_stream_destroy(s); }
  } guard{s};
  std::mt19937_64 rng(seed);
  std::vector<std::byte> host;
  for (size_t i = 0; i < leaves.size(); ++i) {
    const Leaf& l = leaves[i];
    w.bytes += l.size;
    if (gen == "splitmix64" && l.region) {
      auto r = std::make_shared<DeviceRegion>(DeviceRegion::Uninitialized{}, l.size, device);
      if (lzk_fill_splitmix(s, r->device_ptr(), l.size, seed, i) != LZK_OK) {
        throw DeviceError(std::string("workload fill: ") + lzk_last_error());
      }
      w.tree.set_region(l.path, std::move(r));
      continue;
    }
    host.assign(l.size, std::byte{0});
    if (gen == "splitmix64") {
      fill_splitmix_host(host, seed, i);
    } else {
      fill_mt(host, rng);
    }
    if (l.region) {
      w.tree.set_region(l.path, std::make_shared<DeviceRegion>(host, device));
    } else {
      w.tree.set_blob(l.path, host);
    }
  }
  if (lzk_stream_sync(s) != LZK_OK) throw DeviceError(std::string("workload fill sync: ") + lzk_last_error());
  w.leaves = leaves.size();
  return w;
}

}  // namespace lzckpt
