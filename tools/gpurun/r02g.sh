set -x
free -g > gpurun_out/r02g_free.txt; nproc >> gpurun_out/r02g_free.txt
timeout 2400 python bench.py --config cfg5 --steps 1 --warmup 3 > gpurun_out/r02g_cfg5_4096.json 2> gpurun_out/r02g_cfg5_4096.err; echo "exit $?" >> gpurun_out/r02g_cfg5_4096.err
