mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_flux.py -x -q 2>&1 | tail -4 > gpurun_out/flux_tests.txt
timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('S2', d['roofline_flux']['flux_ms_avg'], d['value'])" > gpurun_out/ab.txt
