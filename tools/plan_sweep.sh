#!/bin/bash
# T (1024 x 3072 r16) and C2 step time under forced column-tile counts of the
# fused kernel's plan (OCC_V2_NC, experiment knob), back to back (bench.py).
set -u
mkdir -p gpurun_out
o=gpurun_out/plan
for cfg in T C2; do
  for nc in ${NCS:-0 8 10 12 14 16 18 19 20 24 28 32 37}; do
    if [ "$nc" = 0 ]; then unset OCC_V2_NC; else export OCC_V2_NC=$nc; fi
    timeout 120 python bench.py --config $cfg --steps 100 --warmup 10 --no-cpu-baseline --no-e2e --no-target > ${o}_${cfg}_$nc.json 2>/dev/null
    echo "$cfg nc=$nc $(tail -1 ${o}_${cfg}_$nc.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["roofline"]["frac"])' 2>/dev/null)"
  done
done
unset OCC_V2_NC
