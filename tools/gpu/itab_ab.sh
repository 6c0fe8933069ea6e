python -m pytest tests/test_construct_gpu.py tests/test_montecarlo.py -m gpu -q -x > gpurun_out/t21.log 2>&1
echo "table: $(python tools/time_build.py vehicle3d 2>&1 | tail -1)"
echo "notable: $(IMPACT_NO_INIT_TABLE=1 python tools/time_build.py vehicle3d 2>&1 | tail -1)"
echo "table room5d: $(python tools/time_build.py room5d once 2>&1 | tail -1)"
echo "notable room5d: $(IMPACT_NO_INIT_TABLE=1 python tools/time_build.py room5d once 2>&1 | tail -1)"
python tools/row_parity_report.py vehicle3d room5d > gpurun_out/rowrep21.json 2> gpurun_out/rowrep21.err
