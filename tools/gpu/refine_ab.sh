set -x
IMPACT_EXACT=1 python tools/time_build.py vehicle3d > gpurun_out/tb_exact.txt 2>&1
IMPACT_EXACT=0 python tools/time_build.py vehicle3d > gpurun_out/tb_fast.txt 2>&1
IMPACT_EXACT=0 python tools/time_build.py room5d once >> gpurun_out/tb_fast.txt 2>&1
IMPACT_EXACT=1 python tools/time_build.py room5d once >> gpurun_out/tb_exact.txt 2>&1
python tools/row_parity_report.py vehicle3d room5d robot2d_reachavoid bas7d_verify > gpurun_out/rowrep_fast.json 2> gpurun_out/rowrep_fast.err
