for v in head asm head asm; do
  for c in dim14_verify robot2d_reachavoid; do
    echo "$v $(IMP_LIB_PATH=_variants/libimpact_b200_$v.so python tools/time_build.py $c 2>&1 | tail -1)"
  done
done
echo "asm $(IMP_LIB_PATH=_variants/libimpact_b200_asm.so python tools/time_build.py room5d once 2>&1 | tail -1)"
echo "asm $(IMP_LIB_PATH=_variants/libimpact_b200_asm.so python tools/time_build.py bas7d_verify 2>&1 | tail -1)"
IMP_LIB_PATH=_variants/libimpact_b200_asm.so python -m pytest tests/test_construct_gpu.py tests/test_montecarlo.py -m gpu -q -x > gpurun_out/asm_t.log 2>&1; tail -2 gpurun_out/asm_t.log
