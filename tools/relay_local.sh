# Owner-side local DMA time under a forced relay, both helper routes (2 GPUs).
for route in ce kernel; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2952$([ $route = ce ] && echo 1 || echo 2) bench.py --gpus 2 --steps 3 --warmup 3 --relay force --relay-route $route --skip-configs2 --skip-cpu-baseline --skip-streaming --skip-train --skip-e2e > gpurun_out/r2_relay_local_$route.json 2> gpurun_out/r2_relay_local_$route.err
echo rc=$?
python -c "import json; d=json.load(open('gpurun_out/r2_relay_local_$route.json')); print('$route', d['value'], d['relay']['history'])"
done
