// Phase timing of verify-style trials (where does a ~1-3 MB round trip spend time?)
#include <chrono>
#include <cstdio>
#include <cstring>
#include <map>
#include <random>

#include "lzckpt/consolidation.hpp"
#include "lzckpt/engine.hpp"

using namespace lzckpt;
using clk = std::chrono::steady_clock;
static std::map<std::string, double> acc;
struct T {
  const char* n;
  clk::time_point t0 = clk::now();
  ~T() { acc[n] += std::chrono::duration<double>(clk::now() - t0).count(); }
};

int main() {
  std::mt19937_64 rng(5);
  for (int trial = 0; trial < 40; ++trial) {
    ParallelTopology topo{1, 1, 1, 1, 1};
    ModelSpec model;
    model.param_count = 120000;
    model.layer_count = 4;
    auto dir = std::filesystem::temp_directory_path() / ("tp-" + std::to_string(trial));
    std::filesystem::remove_all(dir);
    EngineConfig cfg;
    cfg.checkpoint_root = dir;
    cfg.host_buffer_bytes = 64 << 20;
    cfg.large_leaf_threshold = 16 << 10;
    cfg.copy_channel = ThrottledChannel{0, 1 << 20};
    std::unique_ptr<Engine> eng;
    { T t{"engine_ctor"}; eng = std::make_unique<Engine>(cfg, topo, RankCoord{}); }
    ManifestStore manifest(dir / "manifest.json");
    CommitCoordinator coord(manifest, topo);
    StateTree tree;
    auto plan = plan_checkpoint(topo, model, 1);
    {
      T t{"tree_build"};
      for (size_t i = 0; i < plan.shards(0).size(); ++i) {
        uint64_t left = plan.shards(0)[i].size_bytes;
        for (int k = 0; left; ++k) {
          uint64_t n = std::min<uint64_t>(left, k % 2 ? 3000 : 200000);
          std::vector<std::byte> b(n, std::byte(k));
          tree.set_region("s" + std::to_string(i) + "/w" + std::to_string(k), std::make_shared<DeviceRegion>(b));
          left -= n;
        }
      }
    }
    std::shared_ptr<CaptureTicket> tk;
    { T t{"capture"}; tk = eng->capture(plan, tree, 1); }
    { T t{"barrier"}; eng->update_barrier(tk); }
    {
      T t{"mutate_all"};
      for (auto& l : tree.flatten()) l.region->mutate([](std::span<std::byte> d) { d[0] = std::byte{1}; });
    }
    { T t{"persist"}; eng->wait_persisted(tk); }
    {
      T t{"commit"};
      EngineCommitParticipant p(*eng, plan, tk);
      coord.run_step(1, {&p});
    }
    { T t{"restore"}; auto back = eng->restore(manifest, 1); }
    { T t{"engine_dtor"}; eng.reset(); }
    { T t{"tree_dtor"}; tree = StateTree(); }
    std::filesystem::remove_all(dir);
  }
  for (auto& [k, v] : acc) std::printf("%-12s %8.2f ms/trial\n", k.c_str(), v * 1e3 / 40);
}
