#!/bin/bash
# full GPU tests, then stage timings with and without an env switch ($1)
O=gpurun_out
mkdir -p $O
python -m pytest tests -m gpu -x -q > $O/tg.log 2>&1
rm -f $O/ab_sw.log
bash tools/ab.sh sw "-" "$1"
for E in "-" "$1"; do
  if [ "$E" = "-" ]; then EV=""; else EV="$E"; fi
  echo "== $E cfg1" >> $O/ab_sw.log
  env $EV python bench.py --config cfg1 --steps 20 --warmup 5 --no-extras 2>&1 | grep '^{' | \
    python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d.get("stages_ms"))' >> $O/ab_sw.log
done
