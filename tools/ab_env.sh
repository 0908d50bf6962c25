#!/bin/bash
# A/B timing on the bench configuration: each argument is "label|ENV=.. ENV=..|lib-variant" (run on the GPU box)
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS}"
mkdir -p gpurun_out
for spec in "$@"; do
  IFS='|' read -r label envs var <<< "$spec"
  if [ -z "$var" ]; then L=paper_1912_09238_b200/libipm.so; else L=paper_1912_09238_b200/libipm_$var.so; fi
  env $envs IPM_LIB=$L timeout 300 $B > gpurun_out/ab_$label.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/ab_$label.json').read().strip().splitlines()[-1]); print('$label', round(d['value']), round(d['roofline']['dual_ms_avg'], 2), round(d['roofline_flux']['flux_ms_avg'], 3), round(d['roofline']['algorithmic']['frac'],3))" || tail -3 gpurun_out/ab_$label.json
done
