mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_flux.py -x -q 2>&1 | tail -5 > gpurun_out/flux_tests.txt
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_strip.json 2> gpurun_out/bench_strip.err
IPM_FLUX_KERNEL=strip timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_flux_strip -s 1 -c 1 -o gpurun_out/strip python bench.py --nx 512 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/strip_ncu.log 2>&1
ncu -i gpurun_out/strip.ncu-rep --page raw --csv > gpurun_out/strip_raw.csv 2>/dev/null
ncu -i gpurun_out/strip.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/strip_src.csv 2>/dev/null
rm -f gpurun_out/strip.ncu-rep
