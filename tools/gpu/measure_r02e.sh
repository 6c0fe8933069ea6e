# after the construction index / staging changes
set -x
python -m pytest tests -m gpu -q -x > gpurun_out/e_tests.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/e_smoke.log 2>&1
for c in robot2d_reachavoid bas7d_verify; do
  python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/e_bench_$c.json 2> gpurun_out/e_bench_$c.err
done
python bench.py --config dim14_verify --horizon 200 --steps 2 --warmup 3 > gpurun_out/e_bench_dim14_h200.json 2> gpurun_out/e_bench_dim14.err
python bench.py --config room5d --horizon 200 --steps 2 --warmup 3 > gpurun_out/e_bench_room5d_h200.json 2> gpurun_out/e_bench_room5d.err
python bench.py > gpurun_out/e_bench_vehicle3d.json 2> gpurun_out/e_bench_vehicle3d.err
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/e_bench_ref.json 2> gpurun_out/e_bench_ref.err
