for v in b0 b2; do
  for c in robot2d_reachavoid vehicle3d; do
    echo "$v $(IMP_LIB_PATH=_variants/libimpact_b200_$v.so python tools/time_synth.py $c 2>&1 | tail -1)"
  done
  for c in room5d dim14_verify; do
    echo "$v $(IMP_LIB_PATH=_variants/libimpact_b200_$v.so python tools/time_synth.py $c 100 2>&1 | tail -1)"
  done
done
IMP_LIB_PATH=_variants/libimpact_b200_b2.so python -m pytest tests/test_synthesis_gpu.py tests/test_sharded_gpu.py -m gpu -q -x > gpurun_out/b2_t.log 2>&1; tail -2 gpurun_out/b2_t.log
