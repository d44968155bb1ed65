df -h /tmp | tail -1
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4
df -h /tmp | tail -1
timeout 900 python tools/sweep.py > gpurun_out/sweep_n1_v2.jsonl 2>/dev/null; cat gpurun_out/sweep_n1_v2.jsonl | cut -c1-240
