#!/bin/bash
# tc_pq: one item in TMEM (default) vs two (FPM_TCPQ_HALF)
rm -f gpurun_out/ab_half.log
bash tools/ab.sh half "-" "FPM_TCPQ_HALF=1"
