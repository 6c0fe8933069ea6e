IMPACT_EXACT=0 python tools/time_build.py vehicle3d > gpurun_out/tb3_fast.txt 2>&1
IMPACT_EXACT=0 python tools/time_build.py room5d once >> gpurun_out/tb3_fast.txt 2>&1
IMPACT_EXACT=1 python tools/row_parity_report.py vehicle3d room5d > gpurun_out/rowrep3_exact.json 2> gpurun_out/rowrep3_exact.err
