#!/bin/bash
# quick A/B of dispatch variants on cfg3 (value, dual ms, frac)
run() { python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['roofline']['dual_ms_avg'],1), round(d['roofline']['frac'],4))"; }
echo "default (T2 SF)"; run
echo "T2 direct";       IPM_SUMFACT=0 run
IPM_LIB=paper_1912_09238_b200/libipm_timers.so python tools/phase_timers.py cfg3 256
