#!/bin/bash
# GPU tests, M-Basis phase trace and the PM-Basis / PM-IntBasis bench lines
# (one gpurun call).  usage (under gpurun): bash tools/gpu_mb.sh
O=gpurun_out
mkdir -p $O
python -m pytest tests -m gpu -x -q > $O/tg.log 2>&1
FPM_MBASIS_TRACE=1 python tools/mbasis_trace.py > $O/mt.log 2>&1
for C in cfg4 ib4; do
  python bench.py --config $C --steps 5 --warmup 3 --no-extras 2>&1 | grep "^{"
done > $O/b4.log
