set -x
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_dual_lbfgs_big -s 1 -c 1 -o gpurun_out/r02ai_lbig \
  python bench.py --config cfg5 --nx 256 --hessian lbfgs --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-alt > gpurun_out/r02ai_ncu_lbig.log 2>&1
ncu -i gpurun_out/r02ai_lbig.ncu-rep --page raw --csv > gpurun_out/r02ai_lbig.raw.csv 2>/dev/null
ncu -i gpurun_out/r02ai_lbig.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/r02ai_lbig.source.csv 2>/dev/null
gzip -f gpurun_out/r02ai_lbig.source.csv; rm -f gpurun_out/r02ai_lbig.ncu-rep
timeout 1500 python bench.py --config cfg5 --steps 1 --warmup 3 --no-e2e > gpurun_out/r02ai_bench_cfg5_4096.json 2> gpurun_out/r02ai_bench_cfg5_4096.err
timeout 2400 python tools/steady_diag.py --cfl 0.25 --start 480000 --window 40000 --snap 4000 --out gpurun_out/r02ai_steady_diag_cfl025 > gpurun_out/r02ai_steady_diag_cfl025.log 2>&1
