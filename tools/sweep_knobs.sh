#!/bin/bash
# k_refine throughput under JIT knobs (MINBS, CHUNKS lists) on config subsets.
for cfg in "vehicle3d 2500 600" "room5d 2500 200"; do
for minb in ${MINBS:-4}; do for ch in ${CHUNKS:-1 2}; do
  echo "minb=$minb chunk=$ch"
  IMPACT_REFINE_MINB=$minb IMPACT_NDTR_CHUNK=$ch ./tools/refine_eff.sh "$cfg"
done; done; done
