python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo tests_rc=$? >> gpurun_out/gputests.log
tail -3 gpurun_out/gputests.log
bash tools/sweep_bench.sh > gpurun_out/sweep_bench_stream.log 2>&1
IMP_SWEEP_STREAM=0 bash tools/sweep_bench.sh > gpurun_out/sweep_bench_nostream.log 2>&1
for c in robot2d_reachavoid vehicle3d dim6_mini room5d_mini; do
  IMP_SWEEP_STREAM=0 timeout 300 python tools/ab_stream.py $c gpurun_out/ab0_$c.npz
  IMP_SWEEP_STREAM=1 timeout 300 python tools/ab_stream.py $c gpurun_out/ab1_$c.npz
  python tools/ab_cmp.py gpurun_out/ab0_$c.npz gpurun_out/ab1_$c.npz
done > gpurun_out/ab.log 2>&1
cat gpurun_out/sweep_bench_stream.log gpurun_out/sweep_bench_nostream.log gpurun_out/ab.log
