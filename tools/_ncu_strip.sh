mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_flux_strip -s 1 -c 1 -o gpurun_out/strip python bench.py --nx 512 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/strip_ncu.log 2>&1
ncu -i gpurun_out/strip.ncu-rep --page raw --csv > gpurun_out/strip_raw.csv 2>/dev/null
ncu -i gpurun_out/strip.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/strip_src.csv 2>/dev/null
rm -f gpurun_out/strip.ncu-rep
