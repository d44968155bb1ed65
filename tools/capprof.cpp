// capture() host cost on a many-leaf workload (LZCKPT_TRACE=1 prints phases)
#include <chrono>
#include <cstdio>
#include "lzckpt/engine.hpp"
#include "lzckpt/workload.hpp"
using namespace lzckpt;
int main(int argc, char** argv) {
  Workload w = build_workload(argv[1], 0);
  EngineConfig cfg;
  cfg.checkpoint_root = "/tmp/capprof";
  cfg.host_buffer_bytes = w.bytes + w.bytes / 8 + (64 << 20);
  cfg.copy_channel = ThrottledChannel{0, 64 << 20};
  cfg.flush.discard = true;
  cfg.large_leaf_threshold = 1024;
  cfg.snapshot.force_kernel = true;
  Engine eng(cfg, w.topo, w.rank);
  auto plan = plan_checkpoint(w.topo, w.model, w.step);
  for (int r = 0; r < 4; ++r) {
    auto t0 = std::chrono::steady_clock::now();
    auto t = eng.capture(plan, w.tree, 1 + r);
    auto t1 = std::chrono::steady_clock::now();
    eng.update_barrier(t);
    auto t2 = std::chrono::steady_clock::now();
    eng.wait_persisted(t);
    auto t3 = std::chrono::steady_clock::now();
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    std::printf("capture %.1f ms  barrier %.1f ms  release %.1f ms  device %.1f ms  host %.2f GB/s\n", ms(t0, t1),
                ms(t1, t2), ms(t2, t3), eng.transfers().ticket_device_ms(t->id()), t->payload_bytes() / (ms(t0, t2) * 1e-3) / 1e9);
  }
}
