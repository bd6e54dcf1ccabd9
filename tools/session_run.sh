set -u
mkdir -p gpurun_out
o=gpurun_out/s4a
timeout 1200 python -m pytest tests -m gpu -q > ${o}_pytest.log 2>&1; echo "pytest rc=$?"; grep -E "FAILED|passed|failed" ${o}_pytest.log | head
timeout 600 python tools/kappa_ab.py > ${o}_kappa.jsonl 2>&1; cut -c1-230 ${o}_kappa.jsonl
for c in C3 C4; do timeout 600 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['config'], d['ms_per_step'], d['eager_ms_per_step'], d['roofline']['frac'], d['orth'])"; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:occ_step_kernel -c 6 --csv --log-file ${o}_orth.csv python tools/dp_driver.py 3 > /dev/null 2>&1; grep -o '"[0-9]*"$' ${o}_orth.csv | tr '\n' ' '
