set -u
mkdir -p gpurun_out
o=gpurun_out/s3s
timeout 1200 python -m pytest tests -m gpu -q > ${o}_pytest.log 2>&1; echo "pytest rc=$?"; grep -E "FAILED|passed|failed" ${o}_pytest.log | head -20
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file ${o}_launches_C4.csv python bench.py --config C4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu C4 rc=$?"
