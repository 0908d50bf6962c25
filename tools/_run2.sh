mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_flux.py tests/test_gpu_parity.py -x -q 2>&1 | tail -5 > gpurun_out/flux_tests.txt
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_strip.json 2> gpurun_out/bench_strip.err
bash tools/_prof.sh
