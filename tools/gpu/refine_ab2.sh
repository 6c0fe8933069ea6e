IMPACT_EXACT=1 python tools/time_build.py vehicle3d > gpurun_out/tb2_exact.txt 2>&1
IMPACT_EXACT=0 python tools/time_build.py vehicle3d > gpurun_out/tb2_fast.txt 2>&1
IMPACT_EXACT=0 python tools/time_build.py room5d once >> gpurun_out/tb2_fast.txt 2>&1
IMPACT_EXACT=1 python tools/row_parity_report.py vehicle3d room5d > gpurun_out/rowrep2_exact.json 2> gpurun_out/rowrep2_exact.err
python tools/row_parity_report.py vehicle3d room5d > gpurun_out/rowrep2_fast.json 2> gpurun_out/rowrep2_fast.err
