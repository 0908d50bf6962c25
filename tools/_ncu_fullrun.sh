# one ncu capture of the dual kernel in the real-run regime (config 3 at 1024^2, step 12 from the IC)
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none -k regex:k_dual_mma -s 12 -c 1 -o gpurun_out/fr python tools/full_run.py cfg3 --steps 13 > gpurun_out/fr_ncu.log 2>&1
ncu -i gpurun_out/fr.ncu-rep --page raw --csv > gpurun_out/fr_raw.csv 2>/dev/null
rm -f gpurun_out/fr.ncu-rep
