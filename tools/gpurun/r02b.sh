set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "stress or full_run or cfg5 or one_shot" > gpurun_out/r02b_par.log 2>&1; echo "exit $?" >> gpurun_out/r02b_par.log
bash tools/ab_env.sh "fixed_newdiag||" "generic_newdiag|IPM_MMA_SHAPE=generic|" "fixed_olddiag||diagshfl" "generic_olddiag|IPM_MMA_SHAPE=generic|diagshfl" > gpurun_out/r02b_ab.txt 2>&1
