mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none -k regex:k_flux_strip -s 2 -c 1 -o gpurun_out/sc python tools/sc_bench.py --nx 1024 --steps 2 --warmup 1 > gpurun_out/sc_ncu.log 2>&1
ncu -i gpurun_out/sc.ncu-rep --page raw --csv > gpurun_out/sc_raw.csv 2>/dev/null
rm -f gpurun_out/sc.ncu-rep
