B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
IPM_DUAL_KERNEL=mma timeout 300 $B > gpurun_out/m5_w2.json 2>&1
IPM_DUAL_KERNEL=mma IPM_MMA_W=4 timeout 300 $B > gpurun_out/m5_w4.json 2>&1
timeout 300 $B > gpurun_out/m5_group.json 2>&1
