set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_linesearch_status.py tests/test_gpu_partition.py tests/test_gpu_edge.py tests/test_gpu_fullsize.py -q -x > gpurun_out/r02d_par.log 2>&1; echo "exit $?" >> gpurun_out/r02d_par.log
bash tools/ab_env.sh "c3_fixed||" "c3_generic|IPM_MMA_SHAPE=generic|" > gpurun_out/r02d_ab.txt 2>&1
BENCH_ARGS="--config cfg4" bash tools/ab_env.sh "c4_bucket||" "c4_single|IPM_BUCKET=0|" >> gpurun_out/r02d_ab.txt 2>&1
