set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_fullsize.py -q -x > gpurun_out/r02c_par.log 2>&1; echo "exit $?" >> gpurun_out/r02c_par.log
bash tools/ab_env.sh "fixed||" "generic|IPM_MMA_SHAPE=generic|" "fixed_nr1||nr1" > gpurun_out/r02c_ab.txt 2>&1
bash tools/ncu_dual_src.sh r02c
