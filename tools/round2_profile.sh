#!/bin/bash
# Round-2 evidence on one GPU (all outputs into gpurun_out/r2f_*):
#   bench lines (C2 default with T beside it, C3, C4, the reference arm), the
#   ncu launch list of the default bench command, and --set full captures of
#   the fused kernel (C2, T) and the large-shape kernels (phase A / D sweeps,
#   band decompress, DP reconstruction).  Each ncu command runs only after the
#   same command has exited 0 without ncu.
#   gpurun --timeout 2400 -- 'bash tools/round2_profile.sh'
set -u
mkdir -p gpurun_out
o=gpurun_out/r2f
timeout 600 python bench.py > ${o}_bench_n1.json 2> ${o}_bench_n1.err || { echo "bench failed"; tail -5 ${o}_bench_n1.err; exit 1; }
tail -1 ${o}_bench_n1.json | cut -c1-300
for c in C3 C4; do timeout 600 python bench.py --config $c --steps 50 --warmup 5 > ${o}_bench_$c.json 2> ${o}_bench_$c.err; done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > ${o}_bench_ref.json 2> ${o}_bench_ref.err
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-target > /dev/null 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file ${o}_launches_n1.csv \
      python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-target > ${o}_ncu_launches.log 2>&1
echo "launch list rc=$?"
for c in C2 T; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:occ_v2_kernel --launch-skip 5 -c 1 \
      -o ${o}_v2_$c python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-target > ${o}_ncu_$c.log 2>&1
  echo "ncu full $c rc=$?"
done
python tools/big_phase_times.py multi > /dev/null 2>&1 && {
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:occ_step_kernel --launch-skip 0 -c 1 \
      -o ${o}_phaseA_C3 python tools/big_phase_times.py multi > ${o}_ncu_pa.log 2>&1; echo "phase A rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:occ_step_kernel --launch-skip 5 -c 1 \
      -o ${o}_phaseD_C3 python tools/big_phase_times.py multi > ${o}_ncu_pd.log 2>&1; echo "phase D rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:occ_v2_decompress_band --launch-skip 0 -c 2 \
      -o ${o}_decompress_C3 python tools/big_phase_times.py multi > ${o}_ncu_dec.log 2>&1; echo "decompress rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:occ_step_kernel --launch-skip 30 -c 1 \
      -o ${o}_phaseF_C4 python tools/big_phase_times.py multi > ${o}_ncu_pf.log 2>&1; echo "phase F rc=$?"
}
timeout 600 python tools/rank_sweep.py > ${o}_rank_sweep.jsonl 2> ${o}_rank_sweep.err
echo "rank sweep rc=$?"
# gpurun brings back at most 64 MiB: keep the raw metric pages (CSV) of every
# capture and only the C2 report itself (source-level view)
for rep in ${o}_*.ncu-rep; do
  ncu -i $rep --page raw --csv > ${rep%.ncu-rep}.raw.csv 2>/dev/null
  ncu -i $rep --page details --csv > ${rep%.ncu-rep}.details.csv 2>/dev/null
  case $rep in *_v2_C2.ncu-rep) ;; *) rm -f $rep ;; esac
done
ls -la gpurun_out | tail -40
