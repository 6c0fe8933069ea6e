for v in head new2; do
echo "$v: $(IMP_LIB_PATH=_variants/libimpact_b200_$v.so python tools/time_build.py vehicle3d 2>&1 | tail -1)"
echo "$v notab: $(IMPACT_NO_INIT_TABLE=1 IMP_LIB_PATH=_variants/libimpact_b200_$v.so python tools/time_build.py vehicle3d 2>&1 | tail -1)"
echo "$v room5d: $(IMP_LIB_PATH=_variants/libimpact_b200_$v.so python tools/time_build.py room5d once 2>&1 | tail -1)"
done
IMP_LIB_PATH=_variants/libimpact_b200_new2.so python -m pytest tests/test_construct_gpu.py -m gpu -q -x -k "golden" > gpurun_out/t22.log 2>&1
