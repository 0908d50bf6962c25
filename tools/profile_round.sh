#!/bin/bash
# Evidence for profiles/: bench line, ncu launch list of the bench command, --set full captures of the
# dual and flux kernels in the bench configuration (cfg3 1024^2, second launch = first timed step).
# usage (on the box): bash tools/profile_round.sh <tag>
tag=${1:-r01}
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${tag}_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-alt > gpurun_out/${tag}_ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_dual_mma -s 1 -c 1 -o gpurun_out/${tag}_dual \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-alt > gpurun_out/${tag}_ncu_dual.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_flux_ -s 1 -c 1 -o gpurun_out/${tag}_flux \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-alt > gpurun_out/${tag}_ncu_flux.log 2>&1

# keep gpurun_out small (<= 64 MiB merge limit): export the pages we read, drop large reports
for rep in gpurun_out/${tag}_dual gpurun_out/${tag}_flux gpurun_out/${tag}_big; do
  if [ -f $rep.ncu-rep ]; then
    ncu -i $rep.ncu-rep --page raw --csv > $rep.raw.csv 2>/dev/null
    ncu -i $rep.ncu-rep --page source --csv --print-source cuda,sass > $rep.source.csv 2>/dev/null
    gzip -f $rep.source.csv
    sz=$(stat -c %s $rep.ncu-rep); if [ $sz -gt 20000000 ]; then rm -f $rep.ncu-rep; fi
  fi
done
echo done > gpurun_out/${tag}_done
