set -x
python -m pytest tests -m gpu -q > gpurun_out/x_tests.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/x_smoke.log 2>&1
python bench.py > gpurun_out/x_bench_vehicle3d.json 2> gpurun_out/x_bench_vehicle3d.err
python bench.py --config room5d --horizon 200 --steps 2 --warmup 3 > gpurun_out/x_bench_room5d_h200.json 2> gpurun_out/x_bench_room5d.err
python bench.py --config robot2d_reachavoid --steps 3 --warmup 3 > gpurun_out/x_bench_robot2d_reachavoid.json 2> gpurun_out/x_bench_robot2d.err
