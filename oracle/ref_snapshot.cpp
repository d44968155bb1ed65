// ORACLE / TEST INFRASTRUCTURE ONLY — links the UNMODIFIED reference library
// (oracle/_ref/liblzckpt_ref.a, built from /root/reference/proj/core/src by
// oracle/Makefile) and drives its public Engine API on a workload spec:
//
//   capture (engine.cpp:96-231) -> update_barrier (engine.cpp:233-253)
//   -> wait_persisted (engine.cpp:255-262) [-> commit_step + restore]
//
// Used (a) to generate golden fixtures / digests for the parity tests,
// (b) as the CPU reference arm of bench.py (`--impl reference`).
//
// usage: ref_snapshot --spec F [--spec F2 ...] --root DIR [--threshold N]
//          [--chunk N] [--pool N] [--fsync 0|1] [--repeat K] [--digest 0|1]
//          [--restore 0|1] [--mode engine|transfer]
// Prints one JSON object on stdout.
#include <chrono>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <map>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "lzckpt/checksum.hpp"
#include "lzckpt/engine.hpp"
#include "lzckpt/errors.hpp"
#include "lzckpt/format.hpp"
#include "lzckpt/manifest.hpp"
#include "lzckpt/topology.hpp"
#include "lzckpt/transfer_engine.hpp"
#include "workload_spec.hpp"

using namespace lzckpt;
namespace fs = std::filesystem;
using clk = std::chrono::steady_clock;

namespace {

struct Opts {
  std::vector<std::string> specs;
  fs::path root = "/tmp/lzk_ref";
  uint64_t threshold = 1ull << 20;
  uint64_t chunk = 64ull << 20;
  uint64_t pool = 0;  // 0: payload of one step + slack
  bool fsync = false;
  int repeat = 1;
  bool digest = true;
  bool restore = false;
  std::string mode = "engine";
  bool keep_last = false;  // delete each step's directory once the next persisted
};

double secs(clk::time_point a, clk::time_point b) {
  return std::chrono::duration<double>(b - a).count();
}

uint64_t file_fnv(const fs::path& p, uint64_t* len) {
  std::ifstream in(p, std::ios::binary);
  Fnv64 h;
  std::vector<char> buf(1 << 20);
  uint64_t n = 0;
  while (in.read(buf.data(), buf.size()) || in.gcount() > 0) {
    h.update(buf.data(), size_t(in.gcount()));
    n += uint64_t(in.gcount());
  }
  *len = n;
  return h.digest();
}

struct RankResult {
  std::string json;
};

std::string run_rank(const Opts& o, const wspec::Spec& s, const std::string& spec_name) {
  ParallelTopology topo{s.dp, s.pp, s.tp, s.gpn, s.nodes};
  RankCoord rank{s.rdp, s.rpp, s.rtp};
  ModelSpec model;
  model.param_count = s.param_count;
  model.layer_count = s.layer_count;
  model.bytes_per_param_model = s.bpp_model;
  model.bytes_per_param_optimizer = s.bpp_opt;

  std::vector<std::vector<std::byte>> bytes;
  auto g0 = clk::now();
  wspec::generate(s, bytes);
  auto g1 = clk::now();

  StateTree tree;
  std::map<std::string, std::pair<bool, const std::vector<std::byte>*>> image;
  for (size_t i = 0; i < s.leaves.size(); ++i) {
    const auto& l = s.leaves[i];
    if (l.region) {
      tree.set_region(l.path, std::make_shared<DeviceRegion>(bytes[i]));
    } else {
      tree.set_blob(l.path, bytes[i]);
    }
    image[l.path] = {l.region, &bytes[i]};
  }
  uint64_t total = tree.total_leaf_bytes();

  char head[512];
  std::string out;
  if (o.mode == "transfer") {
    // TransferEngine alone (transfer_engine.cpp:51-174), no flush consumer.
    HostBufferPool pool(total + 4096);
    TransferEngine te(pool, ThrottledChannel{0.0, o.chunk});
    Segment seg = pool.reserve(total, 1);
    std::vector<std::shared_ptr<CopyTask>> tasks;
    uint64_t dst = 0;
    size_t nreg = 0;
    for (const auto& leaf : tree.flatten()) {
      auto t = std::make_shared<CopyTask>();
      t->source.region = leaf.region;
      t->source.host_blob = leaf.blob;
      t->length = leaf.size;
      t->segment_id = seg.id;
      t->dst_offset = dst;
      dst += leaf.size;
      tasks.push_back(t);
      ++nreg;
    }
    tasks.back()->final_for_segment = true;
    auto t0 = clk::now();
    te.submit_copies(1, tasks);
    te.wait_pending(1);
    auto t1 = clk::now();
    std::snprintf(head, sizeof head,
                  "{\"spec\":\"%s\",\"mode\":\"transfer\",\"bytes\":%llu,\"tasks\":%zu,"
                  "\"seconds\":%.6f,\"gbps\":%.4f}",
                  spec_name.c_str(), (unsigned long long)total, nreg, secs(t0, t1),
                  total / secs(t0, t1) / 1e9);
    return head;
  }

  EngineConfig cfg;
  cfg.checkpoint_root = o.root;
  cfg.copy_channel = ThrottledChannel{0.0, o.chunk};
  cfg.flush = FlushConfig{0, o.fsync};
  cfg.large_leaf_threshold = o.threshold;
  // one step's payload (+ per-file metadata slack) unless overridden
  cfg.host_buffer_bytes = o.pool ? o.pool : total + total / 64 + (64ull << 20);
  Engine engine(cfg, topo, rank);
  ManifestStore manifest(o.root / ("manifest-" + std::to_string(flat_rank(topo, rank)) + ".json"));

  out += "{\"spec\":\"" + spec_name + "\",\"leaves\":" + std::to_string(s.leaves.size()) +
         ",\"leaf_bytes\":" + std::to_string(total) + ",\"gen_s\":" + std::to_string(secs(g0, g1)) +
         ",\"steps\":[";
  std::shared_ptr<CaptureTicket> last;
  for (int r = 0; r < o.repeat; ++r) {
    uint64_t step = s.step + uint64_t(r);
    CheckpointPlan plan = plan_checkpoint(topo, model, step);
    auto t0 = clk::now();
    auto ticket = engine.capture(plan, tree, step);
    auto t1 = clk::now();
    engine.update_barrier(ticket);
    auto t2 = clk::now();
    engine.wait_persisted(ticket);
    auto t3 = clk::now();
    std::snprintf(head, sizeof head,
                  "%s{\"step\":%llu,\"payload\":%llu,\"capture_s\":%.6f,\"barrier_s\":%.6f,"
                  "\"persisted_s\":%.6f}",
                  r ? "," : "", (unsigned long long)step,
                  (unsigned long long)ticket->payload_bytes(), secs(t0, t1), secs(t1, t2),
                  secs(t0, t3));
    out += head;
    if (o.keep_last && last) {
      std::error_code ec;
      fs::remove_all(o.root / step_dirname(last->step()) / rank_dirname(rank), ec);
    }
    last = ticket;
  }
  out += "],\"files\":[";
  CommittedStep committed;
  committed.step = last->step();
  bool first = true;
  for (const auto& f : last->shard_files()) {
    uint64_t len = fs::file_size(f);
    uint64_t d = 0;
    if (o.digest) d = file_fnv(f, &len);
    ManifestFileRecord rec;
    rec.relative_path = fs::relative(f, o.root).generic_string();
    rec.length = len;
    rec.digest = d;
    committed.files.push_back(rec);
    std::snprintf(head, sizeof head, "%s{\"path\":\"%s\",\"size\":%llu,\"fnv\":\"%016llx\"}",
                  first ? "" : ",", rec.relative_path.c_str(), (unsigned long long)len,
                  (unsigned long long)d);
    out += head;
    first = false;
  }
  out += "]";
  if (o.restore) {
    manifest.commit_step(committed);
    auto r0 = clk::now();
    StateTree back = engine.restore(manifest, committed.step);
    auto r1 = clk::now();
    bool exact = back.leaf_count() == image.size();
    for (const auto& leaf : back.flatten()) {
      auto it = image.find(leaf.path);
      if (it == image.end() || it->second.first != (leaf.region != nullptr)) {
        exact = false;
        continue;
      }
      if (leaf.region ? leaf.region->clone_bytes() != *it->second.second
                      : *leaf.blob != *it->second.second) {
        exact = false;
      }
    }
    std::snprintf(head, sizeof head, ",\"restore_s\":%.6f,\"restore_exact\":%s", secs(r0, r1),
                  exact ? "true" : "false");
    out += head;
  }
  out += "}";
  return out;
}

}  // namespace

int main(int argc, char** argv) {
  Opts o;
  for (int i = 1; i < argc; ++i) {
    std::string a = argv[i];
    auto next = [&]() -> std::string {
      if (i + 1 >= argc) throw std::runtime_error("missing value for " + a);
      return argv[++i];
    };
    if (a == "--spec") o.specs.push_back(next());
    else if (a == "--root") o.root = next();
    else if (a == "--threshold") o.threshold = std::stoull(next());
    else if (a == "--chunk") o.chunk = std::stoull(next());
    else if (a == "--pool") o.pool = std::stoull(next());
    else if (a == "--fsync") o.fsync = next() == "1";
    else if (a == "--repeat") o.repeat = std::stoi(next());
    else if (a == "--digest") o.digest = next() == "1";
    else if (a == "--restore") o.restore = next() == "1";
    else if (a == "--mode") o.mode = next();
    else if (a == "--keep-last") o.keep_last = next() == "1";
    else {
      std::fprintf(stderr, "unknown arg %s\n", a.c_str());
      return 2;
    }
  }
  try {
    std::vector<wspec::Spec> specs;
    for (const auto& f : o.specs) specs.push_back(wspec::read_spec(f));
    std::vector<std::string> results(specs.size());
    auto t0 = clk::now();
    // One Engine per rank, run concurrently as threads (bench.cpp:259-318 style).
    std::vector<std::thread> th;
    for (size_t i = 0; i < specs.size(); ++i) {
      th.emplace_back([&, i] { results[i] = run_rank(o, specs[i], o.specs[i]); });
    }
    for (auto& t : th) t.join();
    auto t1 = clk::now();
    std::printf("{\"impl\":\"reference-cpu\",\"threads_per_rank\":2,\"wall_s\":%.6f,\"ranks\":[",
                secs(t0, t1));
    for (size_t i = 0; i < results.size(); ++i) std::printf("%s%s", i ? "," : "", results[i].c_str());
    std::printf("]}\n");
  } catch (const std::exception& e) {
    std::printf("{\"error\":\"%s\"}\n", e.what());
    return 1;
  }
  return 0;
}
