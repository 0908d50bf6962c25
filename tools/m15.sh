B="python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e"
for gr in 2 4 6 8; do
  IPM_MMA_GROUPS=$gr timeout 300 $B > gpurun_out/m15_$gr.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/m15_$gr.json').read().strip().splitlines()[-1]); print($gr, round(d['value']), round(d['roofline']['dual_ms_avg'],1))" >> gpurun_out/m15_summary.txt
done
