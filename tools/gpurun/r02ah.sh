set -x
mkdir -p gpurun_out
BENCH_ARGS="--config cfg5 --nx 512 --no-alt" bash tools/ab_bench.sh bignoswz "" chmin1 bignoswz "" chmin1 > gpurun_out/r02ah_ab_cfg5.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02ah_gputests.log 2>&1; echo "exit $?" >> gpurun_out/r02ah_gputests.log
