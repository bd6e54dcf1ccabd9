#!/bin/bash
# A/B of the phase-5 store L2 policy (evict-first vs normal): timing modes and ncu DRAM bytes, T and C2
set -u
mkdir -p gpurun_out
for dbg in 0 1024; do
  OCC_V2_DEBUG=$dbg python tools/timing_modes.py > gpurun_out/r2ac_tm_$dbg.jsonl 2>&1
  for c in C2 T; do
    OCC_V2_DEBUG=$dbg ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      -k regex:occ_v2_kernel --launch-skip 5 -c 3 --csv python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-target \
      > gpurun_out/r2ac_ncu_${c}_$dbg.csv 2>/dev/null
  done
done
