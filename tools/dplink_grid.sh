#!/bin/bash
# factor_comm_us of the C4 DP step's two factor sums over occ_dplink for several
# CTA caps (OCC_DPLINK_GRID), and the NCCL pair beside it, at N = all GPUs.
set -u
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
o=gpurun_out/dlg_n$NG
for g in 16 32 64 148; do
  OCC_DPLINK_GRID=$g timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29675 bench.py --gpus $NG --config C4 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > ${o}_$g.json 2>/dev/null
  echo "grid $g: $(tail -1 ${o}_$g.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["factor_comm"]["factor_comm_us"])')"
done
