#!/bin/bash
# A/B of the warp-team search bucket count (IMP_K5_LOGB_WARP) on the
# configs with warp-team rows.  Arms: new (in-tree), lw6, lw7 (_variants).
for arm in new lw6 lw7; do
  if [ $arm != new ]; then export IMP_LIB_PATH=$PWD/_variants/libimpact_b200_$arm.so; else unset IMP_LIB_PATH; fi
  timeout 300 python bench.py --config robot2d_reachavoid --steps 2 --no-cpu-baseline > gpurun_out/lb_robot_$arm.json 2>/dev/null
  timeout 400 python bench.py --config room5d --horizon 200 --steps 1 --no-cpu-baseline > gpurun_out/lb_room5d_$arm.json 2>/dev/null
done
unset IMP_LIB_PATH
for f in gpurun_out/lb_*.json; do python -c "
import json,sys; d=json.load(open('$f')); r=d['roofline_sweep']
print('$f', 'sweeps/s %.1f' % d['sweeps_per_s'], 'k5_live_ms %.3f' % r['kernel_ms'], 'settled %.3f' % r['settled']['kernel_ms'], 'ph1_ms %.1f' % d['ms_phase1'])"; done
