set -x
mkdir -p gpurun_out
BENCH_ARGS="--no-alt" bash tools/ab_bench.sh "" ldl "" ldl > gpurun_out/r02t_ab_ldl_cfg3.txt 2>&1
BENCH_ARGS="--config cfg4 --no-alt" bash tools/ab_bench.sh "" ldl > gpurun_out/r02t_ab_ldl_cfg4.txt 2>&1
IPM_LIB=paper_1912_09238_b200/libipm_ldl.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_protocol.py tests/test_gpu_fullsize.py tests/test_gpu_linesearch_status.py -q > gpurun_out/r02t_ldl_tests.log 2>&1; echo "exit $?" >> gpurun_out/r02t_ldl_tests.log
timeout 600 python -m pytest tests/test_gpu_flux.py tests/test_gpu_bands.py -q > gpurun_out/r02t_flux_tests.log 2>&1; echo "exit $?" >> gpurun_out/r02t_flux_tests.log
timeout 600 python bench.py --config cfg4 --no-cpu-baseline --no-e2e --no-alt > gpurun_out/r02t_bench_cfg4.json 2>&1
timeout 600 python bench.py --config cfg5 --nx 512 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-alt > gpurun_out/r02t_bench_cfg5_512.json 2>&1
