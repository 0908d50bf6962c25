B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
for v in "" fx2 ""; do
  if [ -z "$v" ]; then L=paper_1912_09238_b200/libipm.so; else L=paper_1912_09238_b200/libipm_$v.so; fi
  IPM_LIB=$L timeout 300 $B > gpurun_out/m16.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/m16.json').read().strip().splitlines()[-1]); print('$v', round(d['value']), round(d['roofline']['dual_ms_avg'],1), round(d['roofline_flux']['flux_ms_avg'],3), round(d['roofline_flux']['frac'],4))" >> gpurun_out/m16_summary.txt
done
