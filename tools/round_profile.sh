#!/bin/bash
# One GPU, two gpurun calls (one ncu tool per call), all output into gpurun_out/:
#   gpurun --timeout 1200 -- 'bash tools/round_profile.sh launches'
#       bench line (N=1), reference arm, then the ncu launch list of the same bench command
#   gpurun --timeout 1200 -- 'bash tools/round_profile.sh full'
#       the bench command without ncu, then one --set full capture of the fused kernel
set -u
mkdir -p gpurun_out
mode=${1:-launches}
timeout 300 python bench.py --steps 50 --warmup 10 > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err || { echo "bench failed"; tail -5 gpurun_out/bench_n1.err; exit 1; }
tail -1 gpurun_out/bench_n1.json
if [ "$mode" = launches ]; then
  timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
  tail -1 gpurun_out/bench_ref.json
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_n1.csv \
      python bench.py --steps 5 --warmup 3 > gpurun_out/ncu_launches.log 2>&1
  echo "launch list rc=$?"
else
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:occ_v2 --launch-skip 3 -c 1 \
      -o gpurun_out/prof_bench_n1 python bench.py --steps 5 --warmup 3 > gpurun_out/ncu_full.log 2>&1
  echo "ncu full rc=$?"
fi
