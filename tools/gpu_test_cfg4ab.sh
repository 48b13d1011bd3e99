#!/bin/bash
# GPU tests, then cfg4 / ib4 with and without an env switch ($1)
O=gpurun_out
mkdir -p $O
python -m pytest tests -m gpu -x -q > $O/tg.log 2>&1
for E in "-" "$1"; do
  if [ "$E" = "-" ]; then EV=""; else EV="$E"; fi
  for C in cfg4 ib4; do
    echo "== $E $C"
    env $EV python bench.py --config $C --steps 5 --warmup 3 --no-extras 2>&1 | grep '^{' | \
      python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d.get("stages_ms"))'
  done
done > $O/ab4.log 2>&1
