B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $B > gpurun_out/m10_a.json 2>&1
IPM_LIB=paper_1912_09238_b200/libipm_u1.so timeout 300 $B > gpurun_out/m10_b.json 2>&1
timeout 300 $B > gpurun_out/m10_c.json 2>&1
IPM_LIB=paper_1912_09238_b200/libipm_u1.so timeout 300 $B > gpurun_out/m10_d.json 2>&1
