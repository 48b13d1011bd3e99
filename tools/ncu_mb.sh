python tools/pmb_T.py 256 > /dev/null 2>&1
PMB_TS=8 ncu --set full --warp-sampling-interval 0 --clock-control none --import-source on -k regex:mbasis_steps -c 2 -o gpurun_out/mb_steps python tools/pmb_T.py 256 > gpurun_out/ncu_mb.log 2>&1
