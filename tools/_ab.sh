# A/B timing of strip-kernel variants (flux_ms_avg at 1024^2)
cd paper_1912_09238_b200
for v in "NPW=4" "NPW=2"; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -shared -I ../include -DIPM_STRIP_$v csrc/ipm_kernels.cu csrc/ipm_api.cu csrc/ipm_mesh.cpp -o libipm.so
  (cd .. && timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['roofline_flux']['flux_ms_avg'])") >> ../gpurun_out/ab.txt
done
