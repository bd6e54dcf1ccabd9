set -u
mkdir -p gpurun_out
o=gpurun_out/s3f
timeout 300 python tools/umma_dp_check.py > ${o}_umma_dp.jsonl 2>&1; echo "umma dp rc=$?"; cut -c1-400 ${o}_umma_dp.jsonl
OCC_LIB=trace timeout 300 python tools/orth_times.py 3072x12288x64 8192x3072x32 > ${o}_orth.jsonl 2>&1; echo "orth rc=$?"; cat ${o}_orth.jsonl | cut -c1-400
timeout 1200 python -m pytest tests -m gpu -q > ${o}_pytest.log 2>&1; echo "pytest rc=$?"; grep -E "FAILED|passed|failed" ${o}_pytest.log | head -20
for c in C4 C3; do timeout 600 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > ${o}_bench_$c.json 2> ${o}_bench_$c.err; echo "bench $c rc=$?"; tail -1 ${o}_bench_$c.json | cut -c1-300; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file ${o}_launches_C4.csv python bench.py --config C4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu C4 rc=$?"
