set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02a_smi.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_linesearch_status.py -q -x > gpurun_out/r02a_new.log 2>&1; echo "exit $?" >> gpurun_out/r02a_new.log
timeout 1800 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/r02a_gpu.log 2>&1; echo "exit $?" >> gpurun_out/r02a_gpu.log
timeout 600 python bench.py > gpurun_out/r02a_bench.json 2> gpurun_out/r02a_bench.err; echo "exit $?" >> gpurun_out/r02a_bench.err
