#!/bin/bash
# e2e (host buffers) medians: default, copies only (FPM_HOST_DIAG=1), serial
for C in cfg2 cfg3; do
  python tools/e2e_one.py $C 15
  FPM_HOST_DIAG=1 python tools/e2e_one.py $C 15 | sed 's/$/ copies-only/'
  FPM_HOST_BLOCKS=1 python tools/e2e_one.py $C 15 | sed 's/$/ serial/'
done > gpurun_out/e2e_ab.log 2>&1
python tools/micro/pcie.py >> gpurun_out/e2e_ab.log 2>&1
