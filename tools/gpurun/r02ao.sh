set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02ao_gputests.log 2>&1; echo "exit $?" >> gpurun_out/r02ao_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02ao_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/r02ao_smoke.log
bash tools/profile_round.sh r02ao
timeout 600 python bench.py --config cfg4 --no-cpu-baseline > gpurun_out/r02ao_bench_cfg4.json 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02ao_ref.json 2>&1
