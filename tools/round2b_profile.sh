#!/bin/bash
# Round-2 (second part) evidence on one GPU, outputs into gpurun_out/r2g_*:
#   the GPU test log; bench lines (C2 default with T beside it, C3, C4, the
#   reference arm); ncu launch lists of the C2, C3 and C4 bench commands;
#   --set full captures of the fused kernel (C2, T) and of the tcgen05
#   per-phase kernels on the C4 bucket (sweep 1, sweep 2, DP reconstruction,
#   orthonormalisation launch).  Each ncu command runs only after the same
#   command has exited 0 without ncu.
#   gpurun --timeout 3000 -- 'bash tools/round2b_profile.sh'
set -u
mkdir -p gpurun_out
o=gpurun_out/${PREFIX:-r2g}
timeout 1200 python -m pytest tests -m gpu -q > ${o}_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 ${o}_pytest_gpu.log
timeout 600 python bench.py > ${o}_bench_n1.json 2> ${o}_bench_n1.err || { echo "bench failed"; tail -5 ${o}_bench_n1.err; }
tail -1 ${o}_bench_n1.json | cut -c1-200
for c in C3 C4; do timeout 600 python bench.py --config $c --steps 50 --warmup 5 > ${o}_bench_$c.json 2> ${o}_bench_$c.err; echo "bench $c rc=$?"; done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > ${o}_bench_ref.json 2> ${o}_bench_ref.err; echo "ref rc=$?"
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-target > /dev/null 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file ${o}_launches_n1.csv \
      python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-target > /dev/null 2>&1
echo "launch list rc=$?"
for c in C3 C4; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file ${o}_launches_$c.csv \
      python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "launch list $c rc=$?"
done
for c in C2 T; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:occ_v2_kernel --launch-skip 5 -c 1 \
      -o ${o}_v2_$c python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-target > ${o}_ncu_$c.log 2>&1
  echo "ncu full $c rc=$?"
done
python tools/dp_driver.py 3 > /dev/null 2>&1 && {
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:umma_sweep_kernel --launch-skip 4 -c 1 \
      -o ${o}_sweep1_C4 python tools/dp_driver.py 3 > ${o}_ncu_s1.log 2>&1; echo "sweep1 rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:umma_sweep_kernel --launch-skip 6 -c 1 \
      -o ${o}_sweep2_C4 python tools/dp_driver.py 3 > ${o}_ncu_s2.log 2>&1; echo "sweep2 rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:umma_recon --launch-skip 2 -c 1 \
      -o ${o}_recon_C4 python tools/dp_driver.py 3 > ${o}_ncu_rc.log 2>&1; echo "recon rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:occ_step_kernel --launch-skip 2 -c 1 \
      -o ${o}_orth_C4 python tools/dp_driver.py 3 > ${o}_ncu_orth.log 2>&1; echo "orth rc=$?"
}
for rep in ${o}_*.ncu-rep; do
  ncu -i $rep --page raw --csv > ${rep%.ncu-rep}.raw.csv 2>/dev/null
  ncu -i $rep --page details --csv > ${rep%.ncu-rep}.details.csv 2>/dev/null
  case $rep in *_v2_C2.ncu-rep|*_recon_C4.ncu-rep) ;; *) rm -f $rep ;; esac
done
ls -la gpurun_out | grep r2g | tail -40
