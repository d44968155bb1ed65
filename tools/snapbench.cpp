// Bisects the D2H snapshot path on a workload spec: raw copy-engine DMAs of
// the same descriptors (one stream, no engine) versus the TransferEngine
// (issuer + completion threads, events per group) versus the full Engine.
//   snapbench <spec> [group_mb] [quantum_mb]
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <memory>
#include <string>
#include <vector>

#include "lzckpt/engine.hpp"
#include "lzckpt/workload.hpp"
#include "lzk_cuda.h"

using namespace lzckpt;
using clk = std::chrono::steady_clock;

static double secs(clk::time_point a, clk::time_point b) { return std::chrono::duration<double>(b - a).count(); }

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: snapbench <spec> [group_mb] [quantum_mb]\n");
    return 2;
  }
  const uint64_t group = (argc > 2 ? std::atoll(argv[2]) : 256) << 20;
  const uint64_t quantum = (argc > 3 ? std::atoll(argv[3]) : 64) << 20;
  const std::string mode = argc > 4 ? argv[4] : "all";  // raw | engine | all (all pins 2 pools)
  Workload w = build_workload(argv[1], 0);
  std::vector<StateTree::FlatLeaf> leaves = w.tree.flatten();
  uint64_t total = 0;
  for (auto& l : leaves) total += l.size;
  std::printf("workload: %zu leaves, %.2f GB\n", leaves.size(), total / 1e9);

  if (mode != "engine") {
  HostBufferPool pool(total + (64 << 20), std::chrono::milliseconds(60000), PoolOptions{true});
  std::byte* base = pool.data();

  // (a) raw DMAs, one per leaf, one stream
  lzk_stream* s = nullptr;
  lzk_stream_create(0, 1, &s);
  lzk_event *e0, *e1;
  lzk_event_create(0, 0, &e0);
  lzk_event_create(0, 0, &e1);
  std::vector<lzk_copy_desc> d;
  uint64_t off = 0;
  for (auto& l : leaves) {
    if (!l.region) continue;
    d.push_back({reinterpret_cast<uint64_t>(l.region->device_ptr()), reinterpret_cast<uint64_t>(base + off), l.size});
    off += l.size;
  }
  for (int r = 0; r < 3; ++r) {
    auto h0 = clk::now();
    lzk_event_record(e0, s);
    lzk_ce_copy_d2h(s, d.data(), uint32_t(d.size()));
    lzk_event_record(e1, s);
    lzk_event_sync(e1);
    float ms = 0;
    lzk_event_elapsed_ms(e0, e1, &ms);
    std::printf("raw DMA per leaf:          device %.2f GB/s  host %.2f GB/s\n", off / (ms * 1e-3) / 1e9,
                off / secs(h0, clk::now()) / 1e9);
  }
  // (a2) raw DMAs split at quantum
  std::vector<lzk_copy_desc> dq;
  for (auto& x : d) {
    for (uint64_t o = 0; o < x.len; o += quantum) dq.push_back({x.src + o, x.dst + o, std::min(quantum, x.len - o)});
  }
  for (int r = 0; r < 2; ++r) {
    lzk_event_record(e0, s);
    lzk_ce_copy_d2h(s, dq.data(), uint32_t(dq.size()));
    lzk_event_record(e1, s);
    lzk_event_sync(e1);
    float ms = 0;
    lzk_event_elapsed_ms(e0, e1, &ms);
    std::printf("raw DMA per quantum piece: device %.2f GB/s (%zu DMAs)\n", off / (ms * 1e-3) / 1e9, dq.size());
  }
  // (a3) raw gather kernel over the same descriptors
  for (int r = 0; r < 2; ++r) {
    lzk_event_record(e0, s);
    lzk_gather_d2h(s, d.data(), uint32_t(d.size()), 16);
    lzk_event_record(e1, s);
    lzk_event_sync(e1);
    float ms = 0;
    lzk_event_elapsed_ms(e0, e1, &ms);
    std::printf("raw gather kernel 16 CTAs: device %.2f GB/s\n", off / (ms * 1e-3) / 1e9);
  }
  lzk_stream_destroy(s);

  // (b) TransferEngine: one segment, one task per leaf
  for (int variant = 0; variant < 2; ++variant) {
    SnapshotOptions so;
    so.group_bytes = group;
    so.force_copy_engine = variant == 0;
    so.force_kernel = variant == 1;
    TransferEngine te(pool, ThrottledChannel{0.0, quantum}, so);
    for (int r = 0; r < 3; ++r) {
      Segment seg = pool.reserve(total, 1);
      std::vector<std::shared_ptr<CopyTask>> tasks;
      uint64_t o2 = 0;
      for (size_t i = 0; i < leaves.size(); ++i) {
        auto t = std::make_shared<CopyTask>();
        t->source.region = leaves[i].region;
        t->source.host_blob = leaves[i].blob;
        t->length = leaves[i].size;
        t->segment_id = seg.id;
        t->dst_offset = o2;
        t->final_for_segment = i + 1 == leaves.size();
        o2 += leaves[i].size;
        tasks.push_back(t);
      }
      auto h0 = clk::now();
      te.submit_copies(100 + r, tasks);
      auto h1 = clk::now();
      te.wait_pending(100 + r);
      auto h2 = clk::now();
      std::printf("TransferEngine %-6s group %llu MB: submit %.2f ms, host %.2f GB/s, device %.2f GB/s\n",
                  variant ? "kernel" : "CE", (unsigned long long)(group >> 20), secs(h0, h1) * 1e3,
                  total / secs(h0, h2) / 1e9, total / (te.ticket_device_ms(100 + r) * 1e-3) / 1e9);
      pool.begin_flush(seg.id);
      pool.release(seg.id);
    }
  }
  }
  // (c) full Engine: capture -> update_barrier -> (discard tier) wait_persisted
  if (mode != "raw") {
    EngineConfig cfg;
    cfg.checkpoint_root = "/tmp/snapbench_ckpt";
    cfg.host_buffer_bytes = total + total / 64 + (256 << 20);
    cfg.copy_channel = ThrottledChannel{0.0, quantum};
    cfg.flush.discard = true;
    cfg.flush.fsync_on_finalize = false;
    cfg.snapshot.group_bytes = group;
    cfg.pool.hugepages = true;
    Engine eng(cfg, w.topo, w.rank);
    CheckpointPlan plan = plan_checkpoint(w.topo, w.model, w.step);
    for (int r = 0; r < 4; ++r) {
      auto h0 = clk::now();
      auto t = eng.capture(plan, w.tree, 10 + r);
      auto h1 = clk::now();
      eng.update_barrier(t);
      auto h2 = clk::now();
      eng.wait_persisted(t);
      std::printf("Engine: capture %.2f ms, host %.2f GB/s, device %.2f GB/s\n", secs(h0, h1) * 1e3,
                  t->payload_bytes() / secs(h0, h2) / 1e9,
                  t->payload_bytes() / (eng.transfers().ticket_device_ms(t->id()) * 1e-3) / 1e9);
    }
  }
  return 0;
}
