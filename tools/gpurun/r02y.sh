set -x
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_dual_big -s 1 -c 1 -o gpurun_out/r02y_big \
  python bench.py --config cfg5 --nx 256 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-alt > gpurun_out/r02y_ncu_big.log 2>&1
ncu -i gpurun_out/r02y_big.ncu-rep --page raw --csv > gpurun_out/r02y_big.raw.csv 2>/dev/null
ncu -i gpurun_out/r02y_big.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/r02y_big.source.csv 2>/dev/null
gzip -f gpurun_out/r02y_big.source.csv; rm -f gpurun_out/r02y_big.ncu-rep
timeout 1200 python bench.py --config cfg5 --steps 1 --warmup 3 --no-e2e > gpurun_out/r02y_bench_cfg5_4096.json 2> gpurun_out/r02y_bench_cfg5_4096.err
timeout 1300 python tools/steady_run.py --pts 274x92 --hessian lbfgs --max-steps 2000000 --max-seconds 1200 --every 50000 > gpurun_out/r02y_steady_274x92_lbfgs.jsonl 2>&1
