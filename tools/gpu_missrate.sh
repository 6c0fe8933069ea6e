#!/bin/bash
# K5a miss rates in real phase loops + launch list of one synthesis.
for c in robot2d_reachavoid vehicle3d room5d_mini dim6_mini; do
  IMP_SWEEP_STATS=1 timeout 300 python tools/ab_stream.py $c /tmp/x.npz
done > gpurun_out/missrate.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_vehicle3d_synth.csv \
  -k regex:'^(?!k_refine|k_mean|k_outer|k_assemble)' \
  python tools/ab_stream.py vehicle3d /tmp/y.npz > gpurun_out/ncu_launch.log 2>&1
cat gpurun_out/missrate.log; tail -2 gpurun_out/ncu_launch.log
