set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_lbfgs.py tests/test_gpu_nested.py -q > gpurun_out/r02m_tests.log 2>&1; echo "exit $?" >> gpurun_out/r02m_tests.log
timeout 600 python tools/lbfgs_diag.py 1024 100 > gpurun_out/r02m_lbfgs_diag.jsonl 2>&1
