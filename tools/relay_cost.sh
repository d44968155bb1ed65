set -x
for route in ce kernel; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2951$([ $route = ce ] && echo 1 || echo 2) bench.py --gpus 2 --steps 3 --warmup 3 --relay force --relay-route $route --skip-configs2 --skip-cpu-baseline --skip-streaming > gpurun_out/r2_relay_cost_$route.json 2> gpurun_out/r2_relay_cost_$route.err
echo rc=$?
done
