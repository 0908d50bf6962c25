set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_lbfgs.py tests/test_gpu_flux.py tests/test_gpu_bands.py tests/test_gpu_fullsize.py tests/test_gpu_partition.py tests/test_gpu_nested.py tests/test_gpu_parity.py -q > gpurun_out/r02r_tests.log 2>&1; echo "exit $?" >> gpurun_out/r02r_tests.log
timeout 600 python bench.py --config cfg4 --no-cpu-baseline --no-e2e > gpurun_out/r02r_bench_cfg4.json 2>&1
timeout 600 python bench.py --config cfg5 --nx 512 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-alt > gpurun_out/r02r_bench_cfg5_512_newton.json 2>&1
timeout 600 python bench.py --config cfg5 --nx 512 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --hessian lbfgs > gpurun_out/r02r_bench_cfg5_512_lbfgs.json 2>&1
timeout 1500 python bench.py --config cfg5 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --hessian lbfgs > gpurun_out/r02r_bench_cfg5_4096_lbfgs.json 2> gpurun_out/r02r_bench_cfg5_4096_lbfgs.err
