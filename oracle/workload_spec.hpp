// ORACLE / TEST INFRASTRUCTURE ONLY.
//
// Workload spec reader + deterministic synthetic byte generators shared by the
// reference driver (ref_snapshot.cpp). The product has its own independent
// reader (paper_2406_10707_b200/csrc/tools); both must agree byte-for-byte,
// which the parity tests check through file digests.
//
// Spec format (text, one directive per line, '#' comments):
//   model <param_count> <layer_count> <bytes_per_param_model> <bytes_per_param_optimizer>
//   topology <dp> <pp> <tp> <gpus_per_node> <node_count>
//   rank <dp> <pp> <tp>
//   step <N>
//   gen splitmix64 <seed> | gen mt19937_64 <seed>
//   leaf <r|b> <path> <size_bytes>          (creation/fill order)
//
// Generators:
//   mt19937_64: one std::mt19937_64(seed) consumed leaf by leaf in spec order,
//     one 64-bit word per 8 bytes, little-endian, a final partial word donates
//     its leading bytes (tests/test_support.hpp:20-31 of
//     the reference uses the same fill).
//   splitmix64: word w of leaf i = mix64(seed ^ (i * 0xD1B54A32D192ED03) +
//     (w + 1) * 0x9E3779B97F4A7C15), same byte packing; counter-based so the
//     GPU can generate it in parallel.
#pragma once

#include <cstdint>
#include <cstring>
#include <fstream>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

namespace wspec {

struct Leaf {
  bool region = true;
  std::string path;
  uint64_t size = 0;
};

struct Spec {
  uint64_t param_count = 0;
  uint32_t layer_count = 1;
  uint32_t bpp_model = 2;
  uint32_t bpp_opt = 12;
  uint32_t dp = 1, pp = 1, tp = 1, gpn = 1, nodes = 1;
  uint32_t rdp = 0, rpp = 0, rtp = 0;
  uint64_t step = 1;
  std::string gen = "splitmix64";
  uint64_t seed = 0;
  std::vector<Leaf> leaves;
};

inline Spec read_spec(const std::string& file) {
  std::ifstream in(file);
  if (!in) throw std::runtime_error("cannot open spec " + file);
  Spec s;
  std::string line;
  while (std::getline(in, line)) {
    if (line.empty() || line[0] == '#') continue;
    std::istringstream ls(line);
    std::string kw;
    ls >> kw;
    if (kw == "model") {
      ls >> s.param_count >> s.layer_count >> s.bpp_model >> s.bpp_opt;
    } else if (kw == "topology") {
      ls >> s.dp >> s.pp >> s.tp >> s.gpn >> s.nodes;
    } else if (kw == "rank") {
      ls >> s.rdp >> s.rpp >> s.rtp;
    } else if (kw == "step") {
      ls >> s.step;
    } else if (kw == "gen") {
      ls >> s.gen >> s.seed;
    } else if (kw == "leaf") {
      Leaf l;
      std::string kind;
      ls >> kind >> l.path >> l.size;
      l.region = kind == "r";
      s.leaves.push_back(l);
    } else {
      throw std::runtime_error("bad spec directive: " + kw);
    }
  }
  return s;
}

inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

inline uint64_t splitmix_word(uint64_t seed, uint64_t leaf, uint64_t word) {
  return mix64((seed ^ (leaf * 0xD1B54A32D192ED03ull)) + (word + 1) * 0x9E3779B97F4A7C15ull);
}

// Fills every leaf, in spec order, into out[i] (resized to the leaf size).
inline void generate(const Spec& s, std::vector<std::vector<std::byte>>& out) {
  out.resize(s.leaves.size());
  if (s.gen == "mt19937_64") {
    std::mt19937_64 rng(s.seed);
    for (size_t i = 0; i < s.leaves.size(); ++i) {
      auto& b = out[i];
      b.resize(s.leaves[i].size);
      uint64_t k = 0, n = b.size();
      for (; k + 8 <= n; k += 8) {
        uint64_t w = rng();
        std::memcpy(b.data() + k, &w, 8);
      }
      if (k < n) {
        uint64_t w = rng();
        std::memcpy(b.data() + k, &w, n - k);
      }
    }
  } else if (s.gen == "splitmix64") {
    for (size_t i = 0; i < s.leaves.size(); ++i) {
      auto& b = out[i];
      b.resize(s.leaves[i].size);
      uint64_t n = b.size(), k = 0, w = 0;
      for (; k + 8 <= n; k += 8, ++w) {
        uint64_t v = splitmix_word(s.seed, i, w);
        std::memcpy(b.data() + k, &v, 8);
      }
      if (k < n) {
        uint64_t v = splitmix_word(s.seed, i, w);
        std::memcpy(b.data() + k, &v, n - k);
      }
    }
  } else {
    throw std::runtime_error("unknown generator " + s.gen);
  }
}

}  // namespace wspec
