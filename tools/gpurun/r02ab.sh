set -x
mkdir -p gpurun_out
timeout 5000 python tools/steady_run.py --hessian lbfgs --max-steps 4000000 --max-seconds 4700 --every 50000 > gpurun_out/r02ab_steady_baseline_mesh_lbfgs.jsonl 2>&1
