# final captures of the two dominant kernels (current code)
bash tools/gpu/ncu_k5_inloop.sh fin vehicle3d 40 3
python tools/ncu_lines.py gpurun_out/k5_fin.ncu-rep sweep.cu 30 0 > gpurun_out/k5_fin_lines.txt 2>&1
IMPACT_DUMP_JIT=1 python tools/prof_build.py vehicle3d 2000 150 > gpurun_out/fin_refine_plain.log 2>&1
cp impact_construct.cu gpurun_out/fin_impact_construct.cu
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_refine -c 1 -o gpurun_out/fin_refine_v3d python tools/prof_build.py vehicle3d 2000 150 > gpurun_out/fin_refine_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/fin_refine_v3d.ncu-rep > gpurun_out/fin_refine_summary.txt 2>&1
python tools/ncu_lines.py gpurun_out/fin_refine_v3d.ncu-rep impact_construct.cu 40 0 > gpurun_out/fin_refine_lines.txt 2>&1
