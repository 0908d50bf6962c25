#!/bin/bash
# Functional check of bench.py's multi-rank path on ONE GPU: 2 and 4 ranks over gloo (host-staged
# halo exchange), each rank a 256^2 block of config 3.  Timings are meaningless (ranks share a GPU);
# the point is the decomposition, halo exchange, max-over-ranks timing and the JSON line.
mkdir -p gpurun_out
for n in 2 4; do
  IPM_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
    --master-addr 127.0.0.1 --master-port $((29500 + n)) bench.py --gpus $n --nx 256 --steps 2 --warmup 3 \
    --no-cpu-baseline > gpurun_out/multirank_$n.json 2> gpurun_out/multirank_$n.err
  echo "n=$n exit $?" >> gpurun_out/multirank_$n.err
done
