B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
./tools/microbench/rsqrt_check > gpurun_out/m9_rsqrt.json 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q > gpurun_out/m9_tests.log 2>&1
timeout 300 $B > gpurun_out/m9_new.json 2>&1
IPM_LIB=paper_1912_09238_b200/libipm_lib.so timeout 300 $B > gpurun_out/m9_old.json 2>&1
