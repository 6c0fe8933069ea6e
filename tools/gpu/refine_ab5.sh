python -m pytest tests/test_construct_gpu.py -q -k "ndtr" > gpurun_out/t5_ndtr.log 2>&1
IMPACT_EXACT=1 python tools/time_build.py vehicle3d > gpurun_out/tb5.txt 2>&1
IMPACT_EXACT=1 python tools/time_build.py room5d once >> gpurun_out/tb5.txt 2>&1
IMPACT_EXACT=1 IMPACT_NDTR_LEGACY=1 python tools/time_build.py vehicle3d once >> gpurun_out/tb5.txt 2>&1
python -m pytest tests -m gpu -q > gpurun_out/t5.log 2>&1
python tools/row_parity_report.py > gpurun_out/rowrep5.json 2> gpurun_out/rowrep5.err
