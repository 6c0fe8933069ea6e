# round-2 measurement set (one GPU): builder lines of the other four BASELINE
# configs, ncu launch list of the default bench, ncu --set full captures of
# k_refine (exact objective) and of one in-loop phase-1 iteration of K5
set -x
for c in robot2d_reachavoid bas7d_verify; do
  python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/m_bench_$c.json 2> gpurun_out/m_bench_$c.err
done
python bench.py --config room5d --horizon 200 --steps 2 --warmup 3 > gpurun_out/m_bench_room5d_h200.json 2> gpurun_out/m_bench_room5d.err
python bench.py --config dim14_verify --horizon 200 --steps 2 --warmup 3 > gpurun_out/m_bench_dim14_h200.json 2> gpurun_out/m_bench_dim14.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/m_launches_v3d.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/m_launches_v3d.log 2>&1
IMPACT_DUMP_JIT=1 python tools/prof_build.py vehicle3d 2000 150 > gpurun_out/m_refine_plain.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_refine -c 1 -o gpurun_out/m_refine_v3d python tools/prof_build.py vehicle3d 2000 150 > gpurun_out/m_refine_ncu.log 2>&1
cp impact_construct.cu gpurun_out/m_impact_construct.cu
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_sweep -s 40 -c 3 -o gpurun_out/m_k5_v3d python tools/prof_phase.py vehicle3d > gpurun_out/m_k5_ncu.log 2>&1
