PREFIX=${PREFIX2:-r2q} bash tools/round2_multi.sh 2
o=gpurun_out/${PREFIX2:-r2q}
CUDA_VISIBLE_DEVICES=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:occ_step_kernel --launch-skip 2 -c 1 -o ${o}_orth_C4 python tools/dp_driver.py 3 > ${o}_ncu_orth.log 2>&1; echo "orth rc=$?"
ncu -i ${o}_orth_C4.ncu-rep --page raw --csv > ${o}_orth_C4.raw.csv 2>/dev/null; ncu -i ${o}_orth_C4.ncu-rep --page details --csv > ${o}_orth_C4.details.csv 2>/dev/null; rm -f ${o}_orth_C4.ncu-rep
