B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q > gpurun_out/m11_tests.log 2>&1
timeout 300 $B > gpurun_out/m11_a.json 2>&1
IPM_LIB=paper_1912_09238_b200/libipm_u1.so timeout 300 $B > gpurun_out/m11_b.json 2>&1
