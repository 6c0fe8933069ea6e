#!/bin/bash
# A/B of the speculative first search level in K5 pass A (IMP_K5_SPEC):
# GPU tests with the default library, then bench lines per config for
# spec=1 (in-tree) and spec=0 (_variants/libimpact_b200_spec0.so).
python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo tests_rc=$? >> gpurun_out/gputests.log
# arms: new = in-tree; any other name = _variants/libimpact_b200_<arm>.so
for arm in new ${ARMS:-spec0}; do
  if [ $arm != new ]; then export IMP_LIB_PATH=$PWD/_variants/libimpact_b200_$arm.so; fi
  timeout 300 python bench.py --config dim14_verify --horizon 200 --steps 1 --no-cpu-baseline > gpurun_out/ab_dim14_$arm.json 2>/dev/null
  timeout 300 python bench.py --config robot2d_reachavoid --steps 2 --no-cpu-baseline > gpurun_out/ab_robot_$arm.json 2>/dev/null
  timeout 400 python bench.py --config vehicle3d --steps 1 --no-cpu-baseline > gpurun_out/ab_v3d_$arm.json 2>/dev/null
done
unset IMP_LIB_PATH
tail -2 gpurun_out/gputests.log
for f in gpurun_out/ab_*.json; do python -c "
import json,sys; d=json.load(open('$f')); r=d['roofline_sweep']
print('$f', 'sweeps/s %.1f' % d['sweeps_per_s'], 'k5_live_ms %.3f' % r['kernel_ms'], 'settled %.3f' % r['settled']['kernel_ms'], 'ph1_ms %.1f' % d['ms_phase1'])"; done
