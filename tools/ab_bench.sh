#!/bin/bash
# A/B timing of library variants on the bench configuration (run on the GPU box):
#   python paper_1912_09238_b200/build.py --variant=x -DSOME_MACRO   # builds libipm_x.so
#   bash tools/ab_bench.sh "" x "" x                                  # "" = the default libipm.so
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS}"
mkdir -p gpurun_out
for v in "$@"; do
  if [ -z "$v" ]; then L=paper_1912_09238_b200/libipm.so; else L=paper_1912_09238_b200/libipm_$v.so; fi
  IPM_LIB=$L timeout 300 $B > gpurun_out/ab.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); print('${v:-default}', round(d['value']), round(d['roofline']['dual_ms_avg'], 2), round(d['roofline_flux']['flux_ms_avg'], 3))"
done
