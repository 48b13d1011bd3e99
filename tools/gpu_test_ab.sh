#!/bin/bash
# full GPU tests, then stage timings of cfg2 / cfg3 / cfg5 (one gpurun call)
O=gpurun_out
mkdir -p $O
python -m pytest tests -m gpu -x -q > $O/tg.log 2>&1
rm -f $O/ab_cur.log
bash tools/ab.sh cur "-"
