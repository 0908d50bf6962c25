set -x
mkdir -p gpurun_out
for ch in 64 16 8 4 32; do
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-alt --e2e-chunks $ch > gpurun_out/r02ak_e2e_chunks_$ch.json 2>&1
done
