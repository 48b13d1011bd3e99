#!/bin/bash
FPM_TCPQ_DBG=32 python tools/tcpq_trace.py cfg2 > gpurun_out/tcpq_trace.log 2>&1
