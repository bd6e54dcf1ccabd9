#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck, initcheck) on the hot-path
# kernels: the fused v2 kernel on C1 (128x256 r4) and T (1024x3072 r16), the
# per-phase path at r = 64 (v1 sweeps + v2 reconstruct), OCC_ORIENT_T, and
# occ_decompress.  Logs into gpurun_out/sanitize_<tool>.log; one summary line each.
set -u
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  log=gpurun_out/sanitize_${tool}.log
  : > $log
  for shape in 128x256x4 1024x3072x16 640x1024x64 ot:1000x264x16; do
    timeout 900 compute-sanitizer --tool $tool --error-exitcode 99 python tools/one_call.py $shape >> $log 2>&1
    echo "tool=$tool shape=$shape rc=$?" >> $log
  done
  grep -E "ERROR SUMMARY|rc=" $log | tr '\n' ' '; echo
done
