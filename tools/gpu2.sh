timeout 1200 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -s 2>&1 | tail -8
