for v in head mflat head mflat; do
  echo "$v $(IMP_LIB_PATH=_variants/libimpact_b200_$v.so python tools/time_build.py bas7d_verify 2>&1 | tail -1)"
  echo "$v $(IMP_LIB_PATH=_variants/libimpact_b200_$v.so python tools/time_build.py robot2d_reachavoid 2>&1 | tail -1)"
done
echo "mflat $(IMP_LIB_PATH=_variants/libimpact_b200_mflat.so python tools/time_build.py vehicle3d 2>&1 | tail -1)"
echo "mflat $(IMP_LIB_PATH=_variants/libimpact_b200_mflat.so python tools/time_build.py room5d once 2>&1 | tail -1)"
echo "mflat $(IMP_LIB_PATH=_variants/libimpact_b200_mflat.so python tools/time_build.py dim14_verify 2>&1 | tail -1)"
IMP_LIB_PATH=_variants/libimpact_b200_mflat.so python -m pytest tests/test_construct_gpu.py tests/test_montecarlo.py -m gpu -q -x > gpurun_out/mflat_t.log 2>&1; tail -2 gpurun_out/mflat_t.log
