#!/bin/bash
# ncu --set full of one K5 sweep launch.  Usage: tools/ncu_sweep.sh TAG CFG [K0 KN]
TAG=$1; shift
python tools/prof_sweep.py "$@" > gpurun_out/plain_sweep_$TAG.log 2>&1 && \
timeout 400 ncu --set full --import-source on --clock-control none -k regex:${KREGEX:-k_sweep} -s ${KSKIP:-1} -c 1 \
  -o gpurun_out/sweep_$TAG python tools/prof_sweep.py "$@" 2 > gpurun_out/ncu_sweep_$TAG.log 2>&1
tail -1 gpurun_out/ncu_sweep_$TAG.log; cat gpurun_out/plain_sweep_$TAG.log
