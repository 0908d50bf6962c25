timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -k "cfg5" > gpurun_out/m12_tests.log 2>&1
timeout 600 python bench.py --config cfg5 --nx 64 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/m12_cfg5.json 2>&1
