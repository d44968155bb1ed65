N=${1:-1}
if [ "$N" = "1" ]; then
  timeout 1200 python tools/sweep.py > gpurun_out/sweep_n1.jsonl 2> gpurun_out/sweep_n1.err
else
  timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29512 \
    tools/sweep.py > gpurun_out/sweep_n$N.jsonl 2> gpurun_out/sweep_n$N.err
fi
echo "rc=$?"; cat gpurun_out/sweep_n$N.jsonl; tail -3 gpurun_out/sweep_n$N.err
