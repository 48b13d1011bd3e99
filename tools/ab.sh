#!/bin/bash
# A/B stage timings of the product configs under env variants (one gpurun call).
# usage: bash tools/ab.sh TAG "ENV1" "ENV2" ...   (ENV "-" = defaults)
set -u
TAG=$1; shift
O=gpurun_out; mkdir -p $O
for E in "$@"; do
  for C in cfg2 cfg3 cfg5; do
    if [ "$E" = "-" ]; then EV=""; else EV="$E"; fi
    echo "== $E $C" >> $O/ab_$TAG.log
    env $EV timeout 300 python bench.py --config $C --steps 10 --warmup 3 --no-extras 2>&1 | \
      python -c 'import json,sys
for l in sys.stdin:
  l=l.strip()
  if l.startswith("{"):
    d=json.loads(l); print(d["ms_per_step"], d.get("stages_ms"))
  else: print(l[:300])' >> $O/ab_$TAG.log
  done
done
