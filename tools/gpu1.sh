set -x
nvidia-smi --query-gpu=name,clocks.sm --format=csv
cd tests/reftests && for t in bin/*; do timeout 300 ./$t > ../../gpurun_out/ref_$(basename $t).log 2>&1; echo "$t rc=$?"; tail -1 ../../gpurun_out/ref_$(basename $t).log; done; cd ../..
timeout 600 python tools/gpu_check.py 2>&1 | tee gpurun_out/gpu_check.log
