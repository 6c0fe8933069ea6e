#!/bin/bash
# Round measurement: GPU tests, smoke, bench (JSON), warm K5 rates, launch
# list of the bench command, ncu --set full of one warm K5 launch.
python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo tests_rc=$? >> gpurun_out/gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
bash tools/sweep_bench.sh > gpurun_out/sweep_bench.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_bench.csv python bench.py > gpurun_out/ncu_launch_bench.log 2>&1
KSKIP=4 bash tools/ncu_sweep.sh veh vehicle3d 0 2000 > gpurun_out/ncu_sweep_veh.out 2>&1
tail -3 gpurun_out/gputests.log; cat gpurun_out/smoke.log gpurun_out/bench.json gpurun_out/sweep_bench.log
