set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_flux.py -q -k "farfield or cfg4 or tri or warp" > gpurun_out/r02an_farfield_tests.log 2>&1; echo "exit $?" >> gpurun_out/r02an_farfield_tests.log
timeout 200 python tools/steady_run.py --pts 137x46 --farfield --max-seconds 150 --every 10000 > gpurun_out/r02an_steady_137x46_farfield.jsonl 2>&1
timeout 1300 python tools/steady_run.py --farfield --hessian lbfgs --max-seconds 1200 --every 5000 > gpurun_out/r02an_steady_548x183_farfield_lbfgs.jsonl 2>&1
