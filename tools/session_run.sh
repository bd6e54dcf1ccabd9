set -u
mkdir -p gpurun_out
o=gpurun_out/s3l
OCC_LIB=trace timeout 300 python tools/orth_times.py 3072x12288x64 8192x3072x32 > ${o}_orth.jsonl 2>&1; echo "orth rc=$?"; sed -n '1,2p;5,6p' ${o}_orth.jsonl | cut -c1-500
timeout 900 python -m pytest tests -m gpu -q -x > ${o}_pytest.log 2>&1; echo "pytest rc=$?"; grep -E "FAILED|passed|failed" ${o}_pytest.log | head -20
timeout 600 python bench.py --config C4 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > ${o}_bench_C4.json 2> ${o}_bench_C4.err; echo "bench rc=$?"; tail -1 ${o}_bench_C4.json | cut -c180-260
timeout 600 ncu --set full --import-source on --clock-control none -k regex:umma_recon --launch-skip 2 -c 1 -o ${o}_recon python tools/dp_driver.py 3 > ${o}_ncu_recon.log 2>&1; echo "ncu recon rc=$?"
for rep in ${o}_*.ncu-rep; do ncu -i $rep --page raw --csv > ${rep%.ncu-rep}.raw.csv 2>/dev/null; ncu -i $rep --page source --csv --print-source sass > ${rep%.ncu-rep}.sass.csv 2>/dev/null; done
