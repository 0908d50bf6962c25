set -x
bash tools/ab_env.sh "c3_fixed||" "c3_unroll||unroll" > gpurun_out/r02e_ab.txt 2>&1
bash tools/ncu_dual_src.sh r02e
