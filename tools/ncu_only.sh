#!/bin/bash
# ncu --set full of every kernel of one product of CFG (one gpurun call per CFG:
# the merged gpurun_out/ must stay under 64 MiB).  usage: bash tools/ncu_only.sh CFG TAG [COUNT]
set -u
CFG=$1; TAG=$2; CNT=${3:-4}
O=gpurun_out
C="python tools/run_one.py $CFG 1"
$C > $O/plain_${CFG}_$TAG.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:"ntt_|pointwise|tc_|crt_" -c $CNT \
    -o $O/full_${CFG}_$TAG $C > $O/ncu_full_${CFG}_$TAG.log 2>&1
ls -la $O
