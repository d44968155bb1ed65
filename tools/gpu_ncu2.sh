CMD="python bench.py --layers 4 --steps 2 --warmup 3 --skip-train --skip-e2e --skip-streaming --skip-cpu-baseline"
$CMD > gpurun_out/bench_small.json 2> gpurun_out/bench_small.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:lzk_gather -c 400 --csv \
    --log-file gpurun_out/bench_launches.csv $CMD > gpurun_out/ncu_bench.log 2>&1; echo "ncu rc=$?"
tail -1 gpurun_out/bench_small.json | cut -c1-400
