#!/bin/bash
# ncu --set full of k_refine on a vehicle3d subset (12 states), JIT source
# dumped for source correlation.  Usage: tools/ncu_refine.sh TAG [CFG K0 KN]
TAG=$1; CFG=${2:-vehicle3d}; K0=${3:-2500}; KN=${4:-12}
export IMPACT_DUMP_JIT=1
python tools/prof_build.py $CFG $K0 $KN > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 450 ncu --set full --import-source on --clock-control none -k regex:k_refine -c 1 \
  -o gpurun_out/refine_$TAG python tools/prof_build.py $CFG $K0 $KN > gpurun_out/ncu_$TAG.log 2>&1
tail -1 gpurun_out/ncu_$TAG.log; cp impact_construct.cu gpurun_out/impact_construct_$TAG.cu
