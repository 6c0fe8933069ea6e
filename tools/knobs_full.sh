#!/bin/bash
# k_refine on FULL benchmark builds under JIT knob combos "MINB:CHUNK:INST"
# (IMPACT_REFINE_MINB, IMPACT_NDTR_CHUNK, IMPACT_INST_SMEM).
CFG=${CFG:-vehicle3d}
for combo in ${COMBOS:-4:1:0 5:1:0 4:1:1 5:1:1}; do
  IFS=: read minb ch inst <<< "$combo"
  echo -n "minb=$minb chunk=$ch inst_smem=${inst:-0}  "
  IMPACT_REFINE_MINB=$minb IMPACT_NDTR_CHUNK=$ch IMPACT_INST_SMEM=${inst:-0} \
    timeout 300 python tools/time_build.py $CFG once 2>&1 | tail -1 | \
    grep -o "ms_refine=[0-9.]*\|evals/s .*" | tr '\n' ' '
  echo
done
