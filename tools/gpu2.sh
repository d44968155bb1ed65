timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "reference_engine" 2>&1 | tail -30
