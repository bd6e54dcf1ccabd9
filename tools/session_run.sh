set -u
mkdir -p gpurun_out
o=gpurun_out/s4f
timeout 300 python tools/umma_acc.py OCC_UMMA=1 > ${o}_acc.jsonl 2>&1; cut -c1-220 ${o}_acc.jsonl
SHAPE=3072x12288x64 timeout 300 python tools/umma_acc.py OCC_UMMA=1 > ${o}_acc64.jsonl 2>&1; cut -c1-220 ${o}_acc64.jsonl
timeout 1200 python -m pytest tests -m gpu -q > ${o}_pytest.log 2>&1; echo "pytest rc=$?"; grep -E "FAILED|passed|failed" ${o}_pytest.log | head
for at in 1 0; do for c in C3 C4; do OCC_UMMA_ATMEM=$at timeout 600 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('at=$at', d['config']['config'], d['ms_per_step'], d['roofline']['frac'])"; done; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:umma_sweep -c 8 --csv --log-file ${o}_sw.csv python tools/dp_driver.py 2 > /dev/null 2>&1; grep -o '"[0-9]*"$' ${o}_sw.csv | tr '\n' ' '
