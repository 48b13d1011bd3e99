#!/bin/bash
# One profiling call on a B200 box: bench lines, the launch list of the
# default bench command, and --set full captures of every kernel of one cfg2
# and one cfg5 product (dram bytes -> profiles/ncu_traffic.json).
# usage (under gpurun): bash tools/prof_round.sh TAG
set -u
TAG=${1:-r01}
O=gpurun_out
mkdir -p $O
[ -f profiles/int8_peak.json ] || python tools/int8_peak.py $O/int8_peak.json > $O/int8_peak.log 2>&1
python bench.py > $O/bench_cfg2_$TAG.log 2>&1
python bench.py --config cfg5 --steps 5 --warmup 3 --no-extras > $O/bench_cfg5_$TAG.log 2>&1
CMD="python bench.py --steps 3 --warmup 3 --no-extras"
$CMD > $O/plain_$TAG.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/launches_cfg2_$TAG.csv $CMD > $O/ncu_launch_$TAG.log 2>&1
C2="python tools/run_one.py cfg2 2"
$C2 > $O/plain2_$TAG.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:"ntt_|pointwise|tc_|crt_|widen|mbasis" -c 4 \
    -o $O/full_cfg2_$TAG $C2 > $O/ncu_full2_$TAG.log 2>&1
C5="python tools/run_one.py cfg5 1"
$C5 > $O/plain5_$TAG.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:"ntt_|pointwise|tc_|crt_|widen|mbasis" -c 4 \
    -o $O/full_cfg5_$TAG $C5 > $O/ncu_full5_$TAG.log 2>&1
echo done
