set -x
mkdir -p gpurun_out
timeout 1600 python tools/steady_run.py --pts 274x92 --hessian lbfgs --max-seconds 1500 --every 20000 > gpurun_out/r02x_steady_274x92_lbfgs.jsonl 2>&1
