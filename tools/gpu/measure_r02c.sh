# refresh after the K5 CTA barrier / grid-constant commit: the five bench
# lines, the sharded world-1 lines, the whole GPU suite, smoke
set -x
python -m pytest tests -m gpu -q -x > gpurun_out/c_tests.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c_smoke.log 2>&1
python bench.py > gpurun_out/c_bench_vehicle3d.json 2> gpurun_out/c_bench_vehicle3d.err
for c in robot2d_reachavoid bas7d_verify; do
  python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/c_bench_$c.json 2> gpurun_out/c_bench_$c.err
done
python bench.py --config room5d --horizon 200 --steps 2 --warmup 3 > gpurun_out/c_bench_room5d_h200.json 2> gpurun_out/c_bench_room5d.err
python bench.py --config dim14_verify --horizon 200 --steps 2 --warmup 3 > gpurun_out/c_bench_dim14_h200.json 2> gpurun_out/c_bench_dim14.err
IMP_BENCH_FORCE_SHARDED=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 3 --warmup 3 --config robot2d_reachavoid --no-cpu-baseline > gpurun_out/c_sh_r2d.json 2> gpurun_out/c_sh_r2d.err
IMP_BENCH_FORCE_SHARDED=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 1 --steps 2 --warmup 3 --config vehicle3d --no-cpu-baseline > gpurun_out/c_sh_v3d.json 2> gpurun_out/c_sh_v3d.err
