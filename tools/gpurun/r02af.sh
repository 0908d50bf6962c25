set -x
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02af_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/r02af_smoke.log
bash tools/profile_round.sh r02af
timeout 600 python bench.py --config cfg4 --no-cpu-baseline > gpurun_out/r02af_bench_cfg4.json 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_dual_big -s 1 -c 1 -o gpurun_out/r02af_big \
  python bench.py --config cfg5 --nx 256 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-alt > gpurun_out/r02af_ncu_big.log 2>&1
ncu -i gpurun_out/r02af_big.ncu-rep --page raw --csv > gpurun_out/r02af_big.raw.csv 2>/dev/null
ncu -i gpurun_out/r02af_big.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/r02af_big.source.csv 2>/dev/null
gzip -f gpurun_out/r02af_big.source.csv; rm -f gpurun_out/r02af_big.ncu-rep
timeout 600 python bench.py --config cfg5 --nx 512 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-alt > gpurun_out/r02af_bench_cfg5_512.json 2>&1
