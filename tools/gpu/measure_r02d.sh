# after the k_refine changes (unified NM point, fused objective, batch 16)
set -x
python -m pytest tests -m gpu -q -x > gpurun_out/d_tests.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/d_smoke.log 2>&1
python bench.py > gpurun_out/d_bench_vehicle3d.json 2> gpurun_out/d_bench_vehicle3d.err
python bench.py --config room5d --horizon 200 --steps 2 --warmup 3 > gpurun_out/d_bench_room5d_h200.json 2> gpurun_out/d_bench_room5d.err
python tools/row_parity_report.py vehicle3d room5d > gpurun_out/d_rowrep.json 2> gpurun_out/d_rowrep.err
