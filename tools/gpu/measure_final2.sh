# after the K5 window change: whole GPU suite, smoke, default bench, dim14 line
set -x
python -m pytest tests -m gpu -q > gpurun_out/y_tests.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/y_smoke.log 2>&1
python bench.py > gpurun_out/y_bench_vehicle3d.json 2> gpurun_out/y_bench_vehicle3d.err
python bench.py --config dim14_verify --horizon 200 --steps 2 --warmup 3 > gpurun_out/y_bench_dim14_h200.json 2> gpurun_out/y_bench_dim14.err
python bench.py --config room5d --horizon 200 --steps 2 --warmup 3 > gpurun_out/y_bench_room5d_h200.json 2> gpurun_out/y_bench_room5d.err
IMP_BENCH_FORCE_SHARDED=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 1 --steps 2 --warmup 3 --config vehicle3d --no-cpu-baseline > gpurun_out/y_sh_v3d.json 2> gpurun_out/y_sh_v3d.err
