#!/bin/bash
# One gpurun call: GPU parity tests, smoke, a bench line, and the ncu launch list of the bench command.
# usage (from the repo root, on the box): bash tools/gpu_check.sh <tag> [tests=1] [ncu=1]
tag=${1:-run}; tests=${2:-1}; ncu=${3:-1}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${tag}_smi.txt 2>&1
if [ "$tests" = 1 ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_gputests.log 2>&1; echo "tests exit $?" >> gpurun_out/${tag}_gputests.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/${tag}_smoke.log
fi
timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo "bench exit $?" >> gpurun_out/${tag}_bench.err
if [ "$ncu" = 1 ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${tag}_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/${tag}_ncu.log 2>&1; echo "ncu exit $?" >> gpurun_out/${tag}_ncu.log
fi
