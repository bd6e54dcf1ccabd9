#!/bin/bash
# Round-2 multi-GPU evidence: GPU tests (incl. the torchrun checks), bench
# lines at N = NG for C2 (PP ring over occ_link), C3 (same) and C4 (DP), the
# N=1 C3 / C4 lines, and mp_check / threed_check logs.   NG = nproc.
set -u
NG=${1:-2}
mkdir -p gpurun_out
o=gpurun_out/${PREFIX:-r2m}_n$NG
python -m pytest tests -m gpu -q > ${o}_pytest.log 2>&1; echo "rc=$?" >> ${o}_pytest.log
for c in C2 C3 C4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port $((29600 + NG)) \
      bench.py --gpus $NG --config $c --steps 100 --warmup 5 --no-e2e > ${o}_bench_$c.json 2> ${o}_bench_$c.err
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port $((29610 + NG)) \
    bench.py --gpus $NG --config C2 --steps 100 --warmup 5 --no-e2e --exchange nccl > ${o}_bench_C2_nccl.json 2> ${o}_bench_C2_nccl.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port $((29620 + NG)) \
    tests/mp_check.py > ${o}_mp_check.jsonl 2> ${o}_mp_check.err
for l in "" "--link"; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port $((29630 + NG)) \
      tests/threed_check.py $l >> ${o}_threed.jsonl 2>> ${o}_threed.err
done
if [ "$NG" -ge 4 ]; then
  for l in "" "--link"; do
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port $((29640 + NG)) \
        tools/run_3d.py $l >> ${o}_run3d.jsonl 2>> ${o}_run3d.err
  done
fi
if [ "$NG" -eq 2 ]; then
  for c in C3 C4; do CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --config $c --steps 50 --warmup 5 > ${o}_bench_${c}_n1.json 2> ${o}_bench_${c}_n1.err; done
fi
ls -la gpurun_out | grep r2m_
