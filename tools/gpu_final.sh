#!/bin/bash
# round-end evidence: GPU tests, smoke, bench lines, launch list and full captures
O=gpurun_out
mkdir -p $O
python -m pytest tests -m gpu -q > $O/final_tests.log 2>&1
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/final_smoke.log 2>&1
bash tools/prof_round.sh ${1:-v9}
