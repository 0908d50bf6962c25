set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02w_gputests.log 2>&1; echo "exit $?" >> gpurun_out/r02w_gputests.log
timeout 300 python tools/sc_bench.py > gpurun_out/r02w_sc_bench.json 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02w_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/r02w_smoke.log
timeout 900 python bench.py > gpurun_out/r02w_bench.json 2> gpurun_out/r02w_bench.err
timeout 600 python bench.py --config cfg5 --nx 512 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --hessian lbfgs > gpurun_out/r02w_bench_cfg5_512_lbfgs.json 2>&1
