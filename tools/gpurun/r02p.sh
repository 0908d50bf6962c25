set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_lbfgs.py tests/test_gpu_partition.py tests/test_gpu_nested.py tests/test_gpu_bands.py -q > gpurun_out/r02p_tests.log 2>&1; echo "exit $?" >> gpurun_out/r02p_tests.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r02p_bench.json 2> gpurun_out/r02p_bench.err
timeout 600 python bench.py --config cfg5 --nx 512 --hessian lbfgs --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02p_bench_cfg5_512_lbfgs.json 2>&1
timeout 600 python bench.py --config cfg5 --nx 512 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-alt > gpurun_out/r02p_bench_cfg5_512_newton.json 2>&1
BENCH_ARGS="--hessian lbfgs" bash tools/ncu_dual_src.sh r02p_lbfgs k_dual_lbfgs
