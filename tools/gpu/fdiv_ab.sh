for v in head fdiv; do
  for c in dim14_verify robot2d_reachavoid bas7d_verify; do
    echo "$v $(IMP_LIB_PATH=_variants/libimpact_b200_$v.so python tools/time_build.py $c 2>&1 | tail -1)"
  done
  echo "$v $(IMP_LIB_PATH=_variants/libimpact_b200_$v.so python tools/time_build.py vehicle3d 2>&1 | tail -1)"
  echo "$v $(IMP_LIB_PATH=_variants/libimpact_b200_$v.so python tools/time_build.py room5d once 2>&1 | tail -1)"
done
IMP_LIB_PATH=_variants/libimpact_b200_fdiv.so python -m pytest tests/test_construct_gpu.py tests/test_montecarlo.py tests/test_fileio.py -m gpu -q -x > gpurun_out/fdiv_t.log 2>&1; tail -2 gpurun_out/fdiv_t.log
