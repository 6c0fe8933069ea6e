# refresh after the adaptive-hint commit: all five bench lines + reference arm
# + launch list of the default bench + the whole GPU suite
set -x
python -m pytest tests -m gpu -q -x > gpurun_out/b_tests.log 2>&1
python bench.py > gpurun_out/b_bench_vehicle3d.json 2> gpurun_out/b_bench_vehicle3d.err
for c in robot2d_reachavoid bas7d_verify; do
  python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/b_bench_$c.json 2> gpurun_out/b_bench_$c.err
done
python bench.py --config room5d --horizon 200 --steps 2 --warmup 3 > gpurun_out/b_bench_room5d_h200.json 2> gpurun_out/b_bench_room5d.err
python bench.py --config dim14_verify --horizon 200 --steps 2 --warmup 3 > gpurun_out/b_bench_dim14_h200.json 2> gpurun_out/b_bench_dim14.err
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/b_bench_ref.json 2> gpurun_out/b_bench_ref.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/b_launches_v3d.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/b_launches_v3d.log 2>&1
