timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -20 > gpurun_out/pytest_gpu.log
tail -6 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
