#!/bin/bash
# Session-3 round-end measurement: GPU tests, smoke, bench lines of all five
# configs, the reference arm, ncu of an in-loop K5 launch (dim14, search
# heavy) and the launch list of a robot2d_reachavoid build + synthesis.
python -m pytest tests -m gpu -q > gpurun_out/gputests.log 2>&1; echo tests_rc=$? >> gpurun_out/gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python bench.py --config robot2d_reachavoid --steps 3 > gpurun_out/bench_robot2d_reachavoid.json 2>/dev/null
timeout 600 python bench.py --config room5d --horizon 200 --steps 1 > gpurun_out/bench_room5d_h200.json 2>/dev/null
timeout 300 python bench.py --config dim14_verify --horizon 200 --steps 2 > gpurun_out/bench_dim14_verify_h200.json 2>/dev/null
timeout 300 python bench.py --config bas7d_verify --steps 2 > gpurun_out/bench_bas7d_verify.json 2>/dev/null
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ref.json 2> gpurun_out/ref.err
python tools/prof_phase.py dim14_verify 12 > gpurun_out/plain_phase_dim14.log 2>&1 && \
timeout 400 ncu --set full --import-source on --clock-control none -k regex:k_sweep -s 6 -c 1 \
  -o gpurun_out/sweep_inloop_dim14 python tools/prof_phase.py dim14_verify 12 > gpurun_out/ncu_inloop.log 2>&1
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_robot2d.csv python tools/prof_phase.py robot2d_reachavoid > gpurun_out/ncu_launch.log 2>&1
tail -2 gpurun_out/gputests.log; cat gpurun_out/smoke.log; tail -1 gpurun_out/ncu_inloop.log gpurun_out/ncu_launch.log
for f in gpurun_out/bench*.json gpurun_out/ref.json; do echo $f; cut -c1-200 $f; done
