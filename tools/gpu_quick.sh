#!/bin/bash
# quick cfg5 measurement: bench line (no extras) + ncu launch list + one full capture of the NTT kernels
O=gpurun_out/${1:-quick}
mkdir -p $O
python bench.py --no-extras > $O/bench.jsonl 2> $O/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-extras > $O/ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:ntt_mma -c 2 -o $O/mma_full \
    python tools/run_one.py cfg5 1 > $O/ncu_full.log 2>&1
echo done > $O/DONE
