set -x
mkdir -p gpurun_out
BENCH_ARGS="--config cfg5 --nx 512 --no-alt" bash tools/ab_bench.sh bignoswz "" bignoswz "" > gpurun_out/r02ag_ab_cfg5_big_swizzle.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -k "cfg5 or Cfg5 or big or bands or protocol" > gpurun_out/r02ag_gputests_cfg5.log 2>&1; echo "exit $?" >> gpurun_out/r02ag_gputests_cfg5.log
