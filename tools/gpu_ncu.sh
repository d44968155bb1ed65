python tools/kernel_profile.py 65536 268435456 2 > gpurun_out/kp_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:lzk_gather -s 1 -c 2 -o gpurun_out/gather_prof_v2 \
    python tools/kernel_profile.py 65536 268435456 2 > gpurun_out/ncu_full2.log 2>&1; echo "full rc=$?"
python tools/kernel_profile.py 65536 1073741824 3 > gpurun_out/kp_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_v2.csv \
    python tools/kernel_profile.py 65536 1073741824 3 > gpurun_out/ncu_launches.log 2>&1; echo "launches rc=$?"
cat gpurun_out/kp_plain.log
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "full bench rc=$?"
cat gpurun_out/bench_full.json; tail -12 gpurun_out/bench_full.err
