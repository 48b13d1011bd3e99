#!/bin/bash
# cfg1 / cfg0 latency with and without the one-group-per-CTA NTT variant
O=gpurun_out; mkdir -p $O
for E in "-" "FPM_NTT_NO_SMALL=1"; do
  for C in cfg1 cfg3 cfg4; do
    if [ "$E" = "-" ]; then EV=""; else EV="$E"; fi
    echo "== $E $C" >> $O/ab_small.log
    env $EV timeout 300 python bench.py --config $C --steps 20 --warmup 5 --no-extras 2>&1 | \
      python -c 'import json,sys
for l in sys.stdin:
  l=l.strip()
  if l.startswith("{"):
    d=json.loads(l); print(d["ms_per_step"], d.get("stages_ms"))
  else: print(l[:300])' >> $O/ab_small.log
  done
done
