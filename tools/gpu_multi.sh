N=${1:-2}
{ nproc; free -g | head -2; nvidia-smi topo -m; df -h / | tail -1; } > gpurun_out/multi_box_$N.txt 2>&1
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus $N --steps 3 --warmup 3 > gpurun_out/bench_n$N.json 2> gpurun_out/bench_n$N.err; echo "bench rc=$?"
cat gpurun_out/multi_box_$N.txt; cat gpurun_out/bench_n$N.json; grep "\[bench\]" gpurun_out/bench_n$N.err | tail -20; tail -5 gpurun_out/bench_n$N.err
