set -x
mkdir -p gpurun_out
bash tools/ab_bench.sh "" bs1 "" bs1 > gpurun_out/r02al_ab_cfg3_backsub1.txt 2>&1
BENCH_ARGS="--config cfg4 --no-alt" bash tools/ab_bench.sh "" bs1 "" bs1 > gpurun_out/r02al_ab_cfg4_backsub1.txt 2>&1
IPM_LIB=paper_1912_09238_b200/libipm_bs1.so timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_protocol.py tests/test_gpu_linesearch_status.py tests/test_gpu_edge.py tests/test_gpu_fullsize.py -q -k "not cfg5_baseline" > gpurun_out/r02al_bs1_tests.log 2>&1; echo "exit $?" >> gpurun_out/r02al_bs1_tests.log
timeout 300 python -m pytest tests/test_gpu_linesearch_status.py -q -k step_host > gpurun_out/r02al_step_host_tests.log 2>&1; echo "exit $?" >> gpurun_out/r02al_step_host_tests.log
