python tools/kernel_profile.py 65536 268435456 2 > gpurun_out/kp_plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:lzk_gather -s 1 -c 2 -o gpurun_out/gather_prof_v3 \
    python tools/kernel_profile.py 65536 268435456 2 > gpurun_out/ncu_full3.log 2>&1; echo "full rc=$?"
python tools/kernel_profile.py 4096 41943040 2 > gpurun_out/kp_plain4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:lzk_gather -s 1 -c 2 -o gpurun_out/gather_prof_v3_4k \
    python tools/kernel_profile.py 4096 41943040 2 > gpurun_out/ncu_full4.log 2>&1; echo "full4k rc=$?"
cat gpurun_out/kp_plain3.log gpurun_out/kp_plain4.log | cut -c1-150
