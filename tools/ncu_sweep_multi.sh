#!/bin/bash
# ncu --set full of the first C K5 launches (cold hints first, then warm).
# Usage: tools/ncu_sweep_multi.sh TAG C CFG [K0 KN]
TAG=$1; C=$2; shift 2
python tools/prof_sweep.py "$@" > gpurun_out/plain_sweep_$TAG.log 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sweep -c $C \
  -o gpurun_out/sweep_$TAG python tools/prof_sweep.py "$@" 2 > gpurun_out/ncu_sweep_$TAG.log 2>&1
tail -1 gpurun_out/ncu_sweep_$TAG.log; cat gpurun_out/plain_sweep_$TAG.log
