#!/bin/bash
# round-2 evidence on one B200 (run after the tests pass):
#  - default bench line (cfg5, with per-config extras), reference arm, cfg2/3/1 lines
#  - ncu launch list of the default bench command
#  - per-stage DRAM traffic of one product per config (profiles/r02_traffic.json)
#  - ncu --set full of the three cfg5 kernels (tensor-core forward NTT, CTA-pair
#    pointwise, inverse NTT) with tensor-pipe / issue / stall metrics
O=gpurun_out/${1:-ev}
mkdir -p $O
lscpu > $O/lscpu.txt 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv > $O/smi.txt 2>&1
python bench.py > $O/bench_cfg5.jsonl 2> $O/bench_cfg5.err
python bench.py --impl reference --steps 3 --warmup 1 > $O/ref_cfg5.jsonl 2> $O/ref_cfg5.err
for C in cfg2 cfg3 cfg1; do
  python bench.py --config $C --no-extras >> $O/bench_other.jsonl 2>> $O/bench_other.err
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/launches_cfg5.csv python bench.py --steps 2 --warmup 1 --no-extras > $O/ncu_launch.log 2>&1
for C in cfg5 cfg2 cfg3 cfg1; do
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
      --csv --log-file $O/traffic_$C.csv python tools/ncu_traffic.py run $C > $O/traffic_$C.log 2>&1
done
ncu --set full --import-source on --clock-control none -k regex:"ntt_mma64_kernel|tc_pair2_kernel|ntt_inv_persist" \
    -c 3 -o $O/cfg5_full python tools/run_one.py cfg5 1 > $O/cfg5_full.log 2>&1
echo done > $O/DONE
