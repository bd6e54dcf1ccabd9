#!/bin/bash
# factor exchange alone over occ_link at N=2 for several CTA caps of the exchange kernel
set -u
mkdir -p gpurun_out
for g in 1 4 8 16 32; do
  OCC_LINK_GRID=$g timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port $((29700 + g)) bench.py --gpus 2 --config C2 --steps 50 --warmup 5 --no-e2e > gpurun_out/r2ae_grid_$g.json 2>/dev/null
done
