#!/bin/bash
# factor_comm_us of the C4 DP step's two factor sums over occ_dplink (link) and
# NCCL at N = 2 and N = all GPUs (4).
set -u
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
for n in 2 $NG; do
  o=gpurun_out/dlh_n$n
  timeout 600 python -m pytest tests -m gpu -q -x -k dplink > ${o}_pytest.log 2>&1; echo "pytest rc=$?"
  for ex in link nccl; do
    OCC_BENCH_DPLINK=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29685 bench.py --gpus $n --config C4 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --exchange $ex > ${o}_$ex.json 2>/dev/null
    echo "n=$n $ex: $(tail -1 ${o}_$ex.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["factor_comm"]["exchange"], d["factor_comm"]["factor_comm_us"])')"
  done
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29695 tests/mp_check.py > gpurun_out/dlh_mp_check.jsonl 2>/dev/null; echo "mp_check rc=$?"; grep -c '"ok": true' gpurun_out/dlh_mp_check.jsonl; grep -c '"ok": false' gpurun_out/dlh_mp_check.jsonl
