set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_lbfgs.py -q -x > gpurun_out/r02l_lbfgs_tests.log 2>&1; echo "exit $?" >> gpurun_out/r02l_lbfgs_tests.log
timeout 600 python bench.py --hessian lbfgs --no-cpu-baseline > gpurun_out/r02l_bench_lbfgs.json 2> gpurun_out/r02l_bench_lbfgs.err; echo "exit $?" >> gpurun_out/r02l_bench_lbfgs.err
timeout 600 python bench.py --hessian lbfgs --config cfg4 --no-cpu-baseline --no-e2e > gpurun_out/r02l_bench_lbfgs_cfg4.json 2>&1
timeout 600 python bench.py --config cfg4 --no-cpu-baseline --no-e2e > gpurun_out/r02l_bench_newton_cfg4.json 2>&1
timeout 300 python tools/phase_timers.py cfg3 512 > gpurun_out/r02l_phase_cfg3.json 2>&1
