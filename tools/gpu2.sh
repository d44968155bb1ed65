timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "4gib or unpaced_mutation_before or rejected" 2>&1 | tail -25
