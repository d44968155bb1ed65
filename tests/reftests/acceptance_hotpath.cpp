// Our driver for the reference's hot-path acceptance criterion 1
// (reference tests/acceptance_main.cpp:86-107, same seeds and bounds):
// 500 randomized honest round trips byte-exact and committed, and >= 95 of
// 100 skip-barrier trials caught torn with none committed, in < 120 s.
// (Criteria 5-10 exercise the discrete-event simulator: out of scope.)
#include <chrono>
#include <cstdio>
#include <filesystem>

#include "lzckpt/verify.hpp"

int main(int argc, char** argv) {
  const std::filesystem::path scratch =
      argc > 1 ? argv[1] : std::filesystem::temp_directory_path() / "lzk-acceptance";
  const auto t0 = std::chrono::steady_clock::now();
  lzckpt::VerifyOptions honest;
  honest.scratch_dir = scratch / "c1-honest";
  honest.trials = 500;
  honest.seed = 20260818;
  const auto h = lzckpt::run_verification(honest);
  lzckpt::VerifyOptions torn = honest;
  torn.scratch_dir = scratch / "c1-torn";
  torn.trials = 100;
  torn.seed = 31337;
  torn.skip_barrier = true;
  const auto t = lzckpt::run_verification(torn);
  const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  const bool ok = h.byte_exact() == 500 && h.committed() == 500 && t.torn_detected() >= 95 && t.committed() == 0 &&
                  secs < 120.0;
  std::printf("criterion  1: %s  %u/500 byte-exact round trips; %u/100 tears caught, %u committed; %.1f s of 120\n",
              ok ? "PASS" : "FAIL", h.byte_exact(), t.torn_detected(), t.committed(), secs);
  std::filesystem::remove_all(scratch);
  return ok ? 0 : 1;
}
