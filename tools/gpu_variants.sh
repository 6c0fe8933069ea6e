#!/bin/bash
# A/B of library variants (tools/variant_build.sh): warm K5 rates and
# in-loop phase rates.  Usage: tools/gpu_variants.sh TAG...
for tag in "$@"; do
  export IMP_LIB_PATH=$PWD/_variants/libimpact_b200_$tag.so
  echo "== $tag"
  for c in "robot2d_reachavoid" "vehicle3d 0 2000" "dim14_verify" "room5d 0 2000"; do
    timeout 300 python tools/prof_sweep.py $c 2>&1 | tail -1
  done
  for c in robot2d_reachavoid vehicle3d; do
    IMP_SWEEP_STATS=1 timeout 300 python tools/ab_stream.py $c /tmp/v_$c.npz 2>&1 | tail -3 | head -1
  done
done
