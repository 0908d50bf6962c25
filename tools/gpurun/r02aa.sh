set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_protocol.py tests/test_gpu_fullsize.py tests/test_gpu_bands.py tests/test_gpu_lbfgs.py -q -k "cfg5 or Cfg5 or bands or fullsize or protocol or fallback" > gpurun_out/r02aa_tests.log 2>&1; echo "exit $?" >> gpurun_out/r02aa_tests.log
timeout 600 python bench.py --config cfg5 --nx 512 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-alt > gpurun_out/r02aa_bench_cfg5_512.json 2>&1
