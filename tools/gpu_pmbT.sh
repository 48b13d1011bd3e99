#!/bin/bash
# PM-Basis (cfg4) time vs leaf order, leaf cap lifted (one gpurun call)
FPM_PMBASIS_TMAX=64 PMB_TS=32,16,12,8 python tools/pmb_T.py > gpurun_out/pmbT.log 2>&1
