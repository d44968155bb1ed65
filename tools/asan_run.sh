# Runs the ASan+UBSan-built reference suites (tools/asan_build.sh) and summarizes
# the reports per suite into gpurun_out/asan_*.log.
cd "$(dirname "$0")/../build_asan/bin" || exit 1
export ASAN_OPTIONS="protect_shadow_gap=0 detect_leaks=0 halt_on_error=0 replace_intrin=0" UBSAN_OPTIONS="print_stacktrace=1"
for t in test_transfer test_flush test_buffer_pool test_engine test_consolidation test_verify_bench; do
  timeout 600 ./$t > ../../gpurun_out/asan_$t.log 2>&1
  echo "$t rc=$? warnings=$(grep -c 'ERROR: AddressSanitizer\|runtime error' ../../gpurun_out/asan_$t.log) $(tail -1 ../../gpurun_out/asan_$t.log | cut -c1-90)"
done
