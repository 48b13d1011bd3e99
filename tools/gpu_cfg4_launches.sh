#!/bin/bash
# launch list of one cfg4 PM-Basis run (per-kernel time sums vs the wall time)
O=gpurun_out
mkdir -p $O
python tools/run_one.py cfg4 1 > $O/plain4.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/launches_cfg4.csv python tools/run_one.py cfg4 1 > $O/ncu4.log 2>&1
