set -x
mkdir -p gpurun_out
for h in newton lbfgs; do
  timeout 900 python tools/full_run.py cfg1 cfg2 cfg3 --hessian $h >> gpurun_out/r02z_full_runs.jsonl 2>&1
  timeout 600 python tools/full_run.py cfg5 --nx 128 --hessian $h >> gpurun_out/r02z_full_runs.jsonl 2>&1
  timeout 300 python tools/full_run.py cfg4 --steps 2000 --hessian $h >> gpurun_out/r02z_full_runs.jsonl 2>&1
done
