#!/bin/bash
# K5 sweep bandwidth on the benchmark shapes (twice each, to see the noise).
for c in "robot2d_reachavoid" "room5d 0 2000" "vehicle3d 0 2000" "dim14_verify" "robot2d_reach" "bas7d_verify"; do
  timeout 300 python tools/prof_sweep.py $c 2>&1 | tail -1
done
