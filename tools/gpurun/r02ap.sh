set -x
mkdir -p gpurun_out
timeout 300 python bench.py --config cfg4 --no-cpu-baseline > gpurun_out/r02ap_bench_cfg4.json 2>&1
timeout 600 python bench.py > gpurun_out/r02ap_bench.json 2> gpurun_out/r02ap_bench.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02ap_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/r02ap_smoke.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r02ap_gputests.log 2>&1; echo "exit $?" >> gpurun_out/r02ap_gputests.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02ap_cfg4_launches.csv \
  python bench.py --config cfg4 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-alt > gpurun_out/r02ap_ncu_launch.log 2>&1
