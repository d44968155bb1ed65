# Round-1 measurement batch (one GPU): full bench, then the ncu launch list
# of a bounded bench command (run plain first), then the FNV bench.
set -x
timeout 1500 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo bench rc=$?
CMD="python bench.py --layers 4 --steps 2 --warmup 3 --skip-train --skip-streaming --skip-cpu-baseline"
$CMD > gpurun_out/final_small.json 2> gpurun_out/final_small.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:lzk_ -c 600 --csv \
    --log-file gpurun_out/final_launches.csv $CMD > gpurun_out/final_ncu.log 2>&1; echo ncu rc=$?
timeout 600 python tools/fnv_bench.py > gpurun_out/final_fnv.jsonl 2> /dev/null; echo fnv rc=$?
