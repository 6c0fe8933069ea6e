#!/bin/bash
# K5 check: GPU tests, warm sweep rates, in-loop phase rates + search rates.
python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo tests_rc=$? >> gpurun_out/gputests.log
tail -3 gpurun_out/gputests.log
bash tools/sweep_bench.sh > gpurun_out/sweep_bench.log 2>&1
for c in robot2d_reachavoid vehicle3d room5d_mini dim6_mini; do
  IMP_SWEEP_STATS=1 timeout 300 python tools/ab_stream.py $c gpurun_out/k5_$c.npz
done > gpurun_out/k5_phase.log 2>&1
cat gpurun_out/sweep_bench.log gpurun_out/k5_phase.log
