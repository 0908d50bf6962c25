set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02ac_smi.txt 2>&1
for rep in 1 2; do
  timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02ac_gputests_$rep.log 2>&1; echo "exit $?" >> gpurun_out/r02ac_gputests_$rep.log
done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02ac_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/r02ac_smoke.log
IPM_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 --steps 2 --warmup 3 --nx 256 --no-e2e > gpurun_out/r02ac_multirank_gloo_2.json 2>&1
IPM_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 --hessian lbfgs --steps 2 --warmup 3 --nx 256 --no-e2e > gpurun_out/r02ac_multirank_gloo_2_lbfgs.json 2>&1
bash tools/profile_round.sh r02ac
IPM_LIB=paper_1912_09238_b200/libipm_prof.so timeout 300 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-alt > gpurun_out/r02ac_strip_prof.txt 2>&1
timeout 600 python bench.py --config cfg4 --no-cpu-baseline --no-e2e --no-alt > gpurun_out/r02ac_cfg4_morton.json 2>&1
IPM_FLUX_INDEX_ORDER=1 timeout 600 python bench.py --config cfg4 --no-cpu-baseline --no-e2e --no-alt > gpurun_out/r02ac_cfg4_index_order.json 2>&1
BENCH_ARGS="--config cfg4 --no-alt" bash tools/ab_bench.sh "" fw3 "" fw3 > gpurun_out/r02ac_ab_fluxwarp_minb3.txt 2>&1
