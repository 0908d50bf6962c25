set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02k_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02k_gputests.log 2>&1; echo "exit $?" >> gpurun_out/r02k_gputests.log
timeout 600 python bench.py > gpurun_out/r02k_bench.json 2> gpurun_out/r02k_bench.err; echo "exit $?" >> gpurun_out/r02k_bench.err
timeout 1700 python tools/steady_run.py --max-seconds 1500 > gpurun_out/r02k_cfg4_steady.jsonl 2>&1; echo "exit $?" >> gpurun_out/r02k_cfg4_steady.jsonl
