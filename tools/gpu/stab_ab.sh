for v in fdiv stab fdiv stab; do
  for c in dim14_verify robot2d_reachavoid bas7d_verify; do
    echo "$v $(IMP_LIB_PATH=_variants/libimpact_b200_$v.so python tools/time_build.py $c 2>&1 | tail -1)"
  done
done
IMP_LIB_PATH=_variants/libimpact_b200_stab.so python -m pytest tests/test_construct_gpu.py tests/test_fullsize_parity_gpu.py -m gpu -q -x -k "robot2d or dim14 or bas7d or golden or rows" > gpurun_out/stab_t.log 2>&1; tail -2 gpurun_out/stab_t.log
