python bench.py > gpurun_out/bench_v3d.json 2> gpurun_out/bench_v3d.err
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref_v3d.json 2> gpurun_out/bench_ref_v3d.err
