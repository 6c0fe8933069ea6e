#!/bin/bash
# Round-end measurement: GPU tests, smoke, default bench, the other
# BASELINE configs' bench lines, warm K5 rates.
python -m pytest tests -m gpu -q > gpurun_out/gputests.log 2>&1; echo tests_rc=$? >> gpurun_out/gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
for c in robot2d_reachavoid room5d bas7d_verify; do
  timeout 900 python bench.py --config $c --steps 1 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
bash tools/sweep_bench.sh > gpurun_out/sweep_bench.log 2>&1
tail -2 gpurun_out/gputests.log; cat gpurun_out/smoke.log gpurun_out/bench.json
for c in robot2d_reachavoid room5d bas7d_verify; do cut -c1-400 gpurun_out/bench_$c.json; tail -2 gpurun_out/bench_$c.err; done
cat gpurun_out/sweep_bench.log
