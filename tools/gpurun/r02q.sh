set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02q_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02q_gputests.log 2>&1; echo "exit $?" >> gpurun_out/r02q_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02q_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/r02q_smoke.log
bash tools/profile_round.sh r02q
BENCH_ARGS="--config cfg4" bash tools/ncu_dual_src.sh r02q_cfg4flux k_flux_warp
