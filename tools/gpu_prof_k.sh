#!/bin/bash
# full ncu capture of one kernel (regex on the function name) of one bench
# configuration; SKIP matching launches are skipped first
# usage: bash tools/gpu_prof_k.sh OUTDIR KERNEL_REGEX CONFIG [COUNT] [SKIP]
O=gpurun_out/$1
mkdir -p $O
ncu --set full --import-source on --clock-control none -k regex:"$2" --launch-skip ${5:-0} \
    -c ${4:-1} -o $O/full python tools/run_one.py $3 1 > $O/ncu_full.log 2>&1
echo done > $O/DONE
