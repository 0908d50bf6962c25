set -x
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report hazard python tools/sanitize_case.py > gpurun_out/r02i_racecheck.log 2>&1; echo "exit $?" >> gpurun_out/r02i_racecheck.log
for c in cfg1 cfg2; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02i_${c}_graph.json 2>&1
  IPM_GRAPH=0 timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02i_${c}_nograph.json 2>&1
done
BENCH_ARGS="--config cfg4" bash tools/ab_env.sh "c4_new2||" "c4_base||base" > gpurun_out/r02i_ab.txt 2>&1
