set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02o_gputests.log 2>&1; echo "exit $?" >> gpurun_out/r02o_gputests.log
timeout 600 python tools/lbfgs_diag.py 1024 100 > gpurun_out/r02o_lbfgs_diag.jsonl 2>&1
timeout 600 python bench.py --hessian lbfgs --no-cpu-baseline > gpurun_out/r02o_bench_lbfgs.json 2> gpurun_out/r02o_bench_lbfgs.err
timeout 600 python bench.py --config cfg4 --no-cpu-baseline --no-e2e > gpurun_out/r02o_bench_cfg4.json 2>&1
IPM_FLUX_SCALAR_PROJ=1 timeout 600 python bench.py --config cfg4 --no-cpu-baseline --no-e2e > gpurun_out/r02o_bench_cfg4_scalarproj.json 2>&1
IPM_BAND_ROWS=64 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r02o_cfg5_launches.csv \
  python bench.py --config cfg5 --nx 512 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r02o_cfg5_ncu.log 2>&1
timeout 1200 python bench.py --config cfg5 --steps 1 --warmup 3 --no-e2e > gpurun_out/r02o_bench_cfg5_4096.json 2> gpurun_out/r02o_bench_cfg5_4096.err
