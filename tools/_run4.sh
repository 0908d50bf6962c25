mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_flux.py tests/test_gpu_parity.py tests/test_gpu_partition.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -3 > gpurun_out/t4.txt
timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('flux_ms', d['roofline_flux']['flux_ms_avg'], d['value'])" >> gpurun_out/t4.txt
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_flux_strip -s 1 -c 1 --csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/t4_ncu.csv 2>/dev/null
