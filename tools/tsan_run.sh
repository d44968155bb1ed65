# Runs the TSAN-built reference suites (tools/tsan_build.sh) and summarizes
# the reports per suite into gpurun_out/tsan_*.log.
cd "$(dirname "$0")/../build_tsan/bin" || exit 1
export TSAN_OPTIONS="halt_on_error=0 second_deadlock_stack=1 report_signal_unsafe=0 suppressions=$(cd ../.. && pwd)/tools/tsan.supp"
for t in test_transfer test_flush test_buffer_pool test_engine test_consolidation test_verify_bench; do
  timeout 600 ./$t > ../../gpurun_out/tsan_$t.log 2>&1
  echo "$t rc=$? warnings=$(grep -c 'WARNING: ThreadSanitizer' ../../gpurun_out/tsan_$t.log) $(tail -1 ../../gpurun_out/tsan_$t.log | cut -c1-90)"
done
