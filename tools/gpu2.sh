timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
timeout 600 python bench.py --layers 4 --steps 2 --warmup 3 --skip-cpu-baseline > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err; echo "bench rc=$?"
tail -5 gpurun_out/pytest_gpu.log; cat gpurun_out/bench_quick.json; tail -8 gpurun_out/bench_quick.err
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "full bench rc=$?"
cat gpurun_out/bench_full.json; tail -12 gpurun_out/bench_full.err
