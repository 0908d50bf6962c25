set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02ae_gputests.log 2>&1; echo "exit $?" >> gpurun_out/r02ae_gputests.log
bash tools/ab_bench.sh head "" blk64 head "" blk64 > gpurun_out/r02ae_ab_cfg3_pairlist.txt 2>&1
BENCH_ARGS="--config cfg4 --no-alt" bash tools/ab_bench.sh head "" head "" > gpurun_out/r02ae_ab_cfg4_pairlist.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_dual_mma -s 1 -c 1 -o gpurun_out/r02ae_dual \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-alt > gpurun_out/r02ae_ncu_dual.log 2>&1
ncu -i gpurun_out/r02ae_dual.ncu-rep --page raw --csv > gpurun_out/r02ae_dual.raw.csv 2>/dev/null
ncu -i gpurun_out/r02ae_dual.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/r02ae_dual.source.csv 2>/dev/null
gzip -f gpurun_out/r02ae_dual.source.csv; rm -f gpurun_out/r02ae_dual.ncu-rep
