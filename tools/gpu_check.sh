#!/bin/bash
# Full check: GPU tests, smoke, default bench, sharded bench path (world 1).
python -m pytest tests -m gpu -q > gpurun_out/gputests.log 2>&1; echo tests_rc=$? >> gpurun_out/gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
IMP_BENCH_FORCE_SHARDED=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 1 --warmup 3 \
  > gpurun_out/sharded1.json 2> gpurun_out/sharded1.err
tail -2 gpurun_out/gputests.log; cat gpurun_out/smoke.log; cut -c1-600 gpurun_out/bench.json; cut -c1-400 gpurun_out/sharded1.json; tail -2 gpurun_out/bench.err
