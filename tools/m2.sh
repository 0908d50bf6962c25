B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $B > gpurun_out/m2_w2.json 2>gpurun_out/m2_w2.err
IPM_MMA_W=4 timeout 300 $B > gpurun_out/m2_w4.json 2>&1
IPM_LIB=paper_1912_09238_b200/libipm_timers.so timeout 300 python tools/phase_timers.py cfg3 256 > gpurun_out/m2_phase_w2.json 2>&1
IPM_MMA_W=4 IPM_LIB=paper_1912_09238_b200/libipm_timers.so timeout 300 python tools/phase_timers.py cfg3 256 > gpurun_out/m2_phase_w4.json 2>&1
