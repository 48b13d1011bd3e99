#!/bin/bash
# one GPU test file (arg), log to gpurun_out/one_test.log
python -m pytest "$1" -m gpu -q > gpurun_out/one_test.log 2>&1
