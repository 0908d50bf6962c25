#!/bin/bash
# ncu --set full capture of ONE k_dual_mma launch in the bench configuration (the first timed step),
# exported to raw + source CSV (gzip) under gpurun_out/<tag>_dual.*  usage: bash tools/ncu_dual_src.sh <tag> [kernel-regex]
tag=${1:-x}; kre=${2:-k_dual_mma}
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:$kre -s 1 -c 1 -o gpurun_out/${tag}_dual \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/${tag}_ncu_dual.log 2>&1
ncu -i gpurun_out/${tag}_dual.ncu-rep --page raw --csv > gpurun_out/${tag}_dual.raw.csv 2>/dev/null
ncu -i gpurun_out/${tag}_dual.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${tag}_dual.source.csv 2>/dev/null
gzip -f gpurun_out/${tag}_dual.source.csv
rm -f gpurun_out/${tag}_dual.ncu-rep
