set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_lbfgs.py -q > gpurun_out/r02aj_lbfgs_tests.log 2>&1; echo "exit $?" >> gpurun_out/r02aj_lbfgs_tests.log
BENCH_ARGS="--config cfg5 --nx 512 --hessian lbfgs --no-alt" bash tools/ab_bench.sh head "" head "" > gpurun_out/r02aj_ab_cfg5_lbfgs_layout.txt 2>&1
timeout 600 python bench.py --config cfg5 --nx 512 --hessian lbfgs --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-alt > gpurun_out/r02aj_bench_cfg5_512_lbfgs.json 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_dual_lbfgs_big -s 1 -c 1 -o gpurun_out/r02aj_lbig \
  python bench.py --config cfg5 --nx 256 --hessian lbfgs --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-alt > gpurun_out/r02aj_ncu_lbig.log 2>&1
ncu -i gpurun_out/r02aj_lbig.ncu-rep --page raw --csv > gpurun_out/r02aj_lbig.raw.csv 2>/dev/null
rm -f gpurun_out/r02aj_lbig.ncu-rep
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02aj_gputests.log 2>&1; echo "exit $?" >> gpurun_out/r02aj_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02aj_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/r02aj_smoke.log
bash tools/profile_round.sh r02aj
timeout 600 python bench.py --config cfg4 --no-cpu-baseline > gpurun_out/r02aj_bench_cfg4.json 2>&1
