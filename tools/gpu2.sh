timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -40 > gpurun_out/pytest_gpu.log
tail -15 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --skip-cpu-baseline --skip-train --skip-streaming --layers 8 > gpurun_out/bench_e2e.json 2> gpurun_out/bench_e2e.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_e2e.json')); print(d['value'], d['e2e'])"
