set -x
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r02h_gpu.log 2>&1; echo "exit $?" >> gpurun_out/r02h_gpu.log
bash tools/ab_env.sh "c3_new||" "c3_base||base" > gpurun_out/r02h_ab.txt 2>&1
BENCH_ARGS="--config cfg4" bash tools/ab_env.sh "c4_new||" "c4_base||base" >> gpurun_out/r02h_ab.txt 2>&1
