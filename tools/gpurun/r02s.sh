set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_lbfgs.py tests/test_gpu_flux.py tests/test_gpu_bands.py tests/test_gpu_nested.py tests/test_gpu_parity.py -q > gpurun_out/r02s_tests.log 2>&1; echo "exit $?" >> gpurun_out/r02s_tests.log
for cfg in cfg3 cfg4; do
  timeout 600 python bench.py --config $cfg --hessian lbfgs --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02s_${cfg}_lbfgs_smem.json 2>&1
  IPM_LBFGS_PAIRS=reg timeout 600 python bench.py --config $cfg --hessian lbfgs --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02s_${cfg}_lbfgs_reg.json 2>&1
done
timeout 600 python bench.py --config cfg4 --no-cpu-baseline --no-e2e --no-alt > gpurun_out/r02s_bench_cfg4.json 2>&1
