set -u
mkdir -p gpurun_out
o=gpurun_out/s3x_n$(nvidia-smi -L | wc -l)
NG=$(nvidia-smi -L | wc -l)
timeout 600 python -m pytest tests -m gpu -q -x -k "dplink or dp_" > ${o}_pytest.log 2>&1; echo "pytest rc=$?"; grep -E "FAILED|passed|failed|Error" ${o}_pytest.log | head
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29655 tests/mp_check.py > ${o}_mp_check.jsonl 2> ${o}_mp_check.err; echo "mp_check rc=$?"; grep dp_link ${o}_mp_check.jsonl | cut -c1-220; tail -3 ${o}_mp_check.err
for ex in link nccl; do timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29665 bench.py --gpus $NG --config C4 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline --exchange $ex > ${o}_bench_C4_$ex.json 2> ${o}_bench_C4_$ex.err; echo "bench $ex rc=$?"; tail -1 ${o}_bench_C4_$ex.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["roofline"]["frac"], json.dumps(d["factor_comm"])[:260])'; done
