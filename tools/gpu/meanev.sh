python bench.py --config bas7d_verify --steps 3 --warmup 3 > gpurun_out/g_bench_bas7d_verify.json 2> gpurun_out/g_bench_bas7d.err
python tools/time_build.py vehicle3d > gpurun_out/g_tb.txt 2>&1
python -m pytest tests/test_construct_gpu.py tests/test_synthesis_gpu.py -m gpu -q -x > gpurun_out/g_tests.log 2>&1
