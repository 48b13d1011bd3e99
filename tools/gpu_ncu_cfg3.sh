#!/bin/bash
# launch list + full capture of one cfg3 product
O=gpurun_out
mkdir -p $O
python tools/run_one.py cfg3 2 > $O/plain3.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/launches_cfg3.csv python tools/run_one.py cfg3 2 > $O/ncu3l.log 2>&1
bash tools/ncu_only.sh cfg3 v9 8 > /dev/null 2>&1
