set -x
cd paper_1912_09238_b200
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -shared -I ../include -DIPM_STRIP_PROF csrc/ipm_kernels.cu csrc/ipm_api.cu csrc/ipm_mesh.cpp -o libipm.so
cd ..
timeout 300 python bench.py --nx 512 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline 2>&1 | grep PROF | sort -t' ' -k4,4n -k2,2n > gpurun_out/prof.txt
