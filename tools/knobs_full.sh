#!/bin/bash
# k_refine on FULL benchmark builds under JIT knob combos
# "MINB:CHUNK:INST:BATCH" (IMPACT_REFINE_MINB, IMPACT_NDTR_CHUNK,
# IMPACT_INST_SMEM, IMPACT_REFINE_BATCH).
CFG=${CFG:-vehicle3d}
for combo in ${COMBOS:-5:1:0:2 4:1:0:2}; do
  IFS=: read minb ch inst batch <<< "$combo"
  echo -n "minb=$minb chunk=$ch inst_smem=${inst:-0} batch=${batch:-2}  "
  IMPACT_REFINE_MINB=$minb IMPACT_NDTR_CHUNK=$ch IMPACT_INST_SMEM=${inst:-0} \
  IMPACT_REFINE_BATCH=${batch:-2} timeout 300 python tools/time_build.py $CFG once 2>&1 | tail -1
done
