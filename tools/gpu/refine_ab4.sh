for t in 0 1; do
IMPACT_NDTR_FAST_TABLE=$t python tools/time_build.py vehicle3d > gpurun_out/tb4_$t.txt 2>&1
IMPACT_NDTR_FAST_TABLE=$t python tools/time_build.py room5d once >> gpurun_out/tb4_$t.txt 2>&1
done
python tools/row_parity_report.py vehicle3d room5d > gpurun_out/rowrep4_fast.json 2> gpurun_out/rowrep4_fast.err
