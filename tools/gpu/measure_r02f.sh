python bench.py --config robot2d_reachavoid --steps 3 --warmup 3 > gpurun_out/f_bench_robot2d_reachavoid.json 2> gpurun_out/f_bench_robot2d.err
python bench.py --config dim14_verify --horizon 200 --steps 2 --warmup 3 > gpurun_out/f_bench_dim14_h200.json 2> gpurun_out/f_bench_dim14.err
python -m pytest tests/test_construct_gpu.py tests/test_fullsize_parity_gpu.py tests/test_fileio.py -m gpu -q -x > gpurun_out/f_tests.log 2>&1
