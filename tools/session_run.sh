set -u
mkdir -p gpurun_out
o=gpurun_out/s4e
timeout 1200 python -m pytest tests -m gpu -q > ${o}_pytest.log 2>&1; echo "pytest rc=$?"; grep -E "FAILED|passed|failed" ${o}_pytest.log | head
for pdl in 1 0; do OCC_V2_PDL=$pdl timeout 600 python bench.py --steps 200 --warmup 10 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); t=d['north_star_target']; print('pdl=$pdl', d['ms_per_step'], d['eager_ms_per_step'], d['roofline']['frac'], t['ms_per_step'], t['eager_ms_per_step'], t['roofline_frac'])"; done
for pdl in 1 0; do OCC_V2_PDL=$pdl python tools/graph_probe.py T; done
