set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_lbfgs.py tests/test_gpu_nested.py -q > gpurun_out/r02n_tests.log 2>&1; echo "exit $?" >> gpurun_out/r02n_tests.log
timeout 600 python tools/lbfgs_diag.py 1024 400 > gpurun_out/r02n_lbfgs_diag.jsonl 2>&1
timeout 600 python bench.py --hessian lbfgs --no-cpu-baseline > gpurun_out/r02n_bench_lbfgs.json 2> gpurun_out/r02n_bench_lbfgs.err
for pts in 40x14 137x46 274x92; do
  timeout 420 python tools/steady_run.py --pts $pts --max-seconds 360 --every 5000 > gpurun_out/r02n_steady_$pts.jsonl 2>&1
done
IPM_BAND_ROWS=64 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r02n_cfg5_launches.csv \
  python bench.py --config cfg5 --nx 512 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r02n_cfg5_ncu.log 2>&1
