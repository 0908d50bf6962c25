set -x
timeout 900 python -m pytest tests/test_gpu_bands.py tests/test_gpu_linesearch_status.py -q -x > gpurun_out/r02f_tests.log 2>&1; echo "exit $?" >> gpurun_out/r02f_tests.log
timeout 900 python bench.py --config cfg5 --nx 1024 --steps 2 --warmup 3 --no-e2e > gpurun_out/r02f_cfg5_1024.json 2> gpurun_out/r02f_cfg5_1024.err; echo "exit $?" >> gpurun_out/r02f_cfg5_1024.err
