# final round-2 record: whole GPU suite, smoke, default bench line, launch list
set -x
python -m pytest tests -m gpu -q > gpurun_out/z_tests.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/z_smoke.log 2>&1
python bench.py > gpurun_out/z_bench_vehicle3d.json 2> gpurun_out/z_bench_vehicle3d.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/z_launches_v3d.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/z_launches_v3d.log 2>&1
