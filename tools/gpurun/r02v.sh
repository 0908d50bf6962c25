set -x
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_dual_lbfgs_big -s 1 -c 1 -o gpurun_out/r02v_lbfgs_big \
  python bench.py --config cfg5 --nx 256 --hessian lbfgs --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r02v_ncu_big.log 2>&1
ncu -i gpurun_out/r02v_lbfgs_big.ncu-rep --page raw --csv > gpurun_out/r02v_lbfgs_big.raw.csv 2>/dev/null
ncu -i gpurun_out/r02v_lbfgs_big.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/r02v_lbfgs_big.source.csv 2>/dev/null
gzip -f gpurun_out/r02v_lbfgs_big.source.csv; rm -f gpurun_out/r02v_lbfgs_big.ncu-rep
timeout 1000 python tools/steady_run.py --newton full --max-seconds 900 --every 5000 > gpurun_out/r02v_cfg4_steady_full.jsonl 2>&1
timeout 800 python tools/steady_run.py --hessian lbfgs --max-seconds 700 --every 5000 > gpurun_out/r02v_cfg4_steady_lbfgs.jsonl 2>&1
