set -x
mkdir -p gpurun_out
for cfg in cfg3 cfg4; do
  timeout 600 python bench.py --config $cfg --hessian lbfgs --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02u_${cfg}_lbfgs_fixed.json 2>&1
  IPM_MMA_SHAPE=generic timeout 600 python bench.py --config $cfg --hessian lbfgs --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02u_${cfg}_lbfgs_generic.json 2>&1
done
timeout 900 python -m pytest tests/test_gpu_lbfgs.py tests/test_gpu_nested.py -q > gpurun_out/r02u_tests.log 2>&1; echo "exit $?" >> gpurun_out/r02u_tests.log
