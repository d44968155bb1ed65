#!/bin/bash
# Round-2 profiling pass (one GPU): gather-kernel parity, aligned + skewed
# class timings, the bench's launch list, and one `ncu --set full` capture of
# lzk_gather_kernel per layout. Every ncu command runs only after the same
# command exited 0 without ncu.
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "gather or kernel" > gpurun_out/r02p_pytest.log 2>&1; echo "pytest rc=$?"
for sz in 65536 65539; do
  timeout 300 python tools/kernel_profile.py $sz 1073741824 3 > gpurun_out/r02p_kp_$sz.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:lzk_gather -s 1 -c 1 \
      -o gpurun_out/r02p_gather_$sz python tools/kernel_profile.py $sz 268435456 2 > gpurun_out/r02p_ncu_$sz.log 2>&1
  echo "class $sz rc=$?"
done
CMD="python bench.py --layers 4 --steps 2 --warmup 3 --skip-train --skip-e2e --skip-streaming --skip-cpu-baseline"
timeout 600 $CMD > gpurun_out/r02p_bench_small.json 2> gpurun_out/r02p_bench_small.err && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:lzk -c 400 --csv \
    --log-file gpurun_out/r02p_bench_launches.csv $CMD > gpurun_out/r02p_ncu_bench.log 2>&1; echo "launch list rc=$?"
tail -1 gpurun_out/r02p_bench_small.json | cut -c1-300
cat gpurun_out/r02p_kp_*.log | cut -c1-200
