#!/bin/bash
# one ncu --set full capture of the dual kernel (first launch after warm-up) at a bench-like size
tag=${1:-x}; nx=${2:-512}; kern=${3:-k_dual}
IPM_DUAL_KERNEL=${4:-mma} timeout 900 ncu --set full --import-source on --clock-control none -k regex:$kern -s 1 -c 1 -o gpurun_out/${tag} \
  python bench.py --nx $nx --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/${tag}_ncu.log 2>&1
echo "ncu exit $?" >> gpurun_out/${tag}_ncu.log
