python -m pytest tests/test_synthesis_gpu.py tests/test_fullsize_gpu.py tests/test_sharded_gpu.py -m gpu -q -x > gpurun_out/t16.log 2>&1
for v in staged exact; do
  for c in robot2d_reachavoid vehicle3d; do
    echo "$v $(IMP_LIB_PATH=_variants/libimpact_b200_$v.so python tools/time_synth.py $c 2>&1 | tail -1)"
  done
  echo "$v $(IMP_LIB_PATH=_variants/libimpact_b200_$v.so python tools/time_synth.py dim14_verify 100 2>&1 | tail -1)"
  echo "$v $(IMP_LIB_PATH=_variants/libimpact_b200_$v.so python tools/time_synth.py room5d 100 2>&1 | tail -1)"
  echo "$v $(IMP_LIB_PATH=_variants/libimpact_b200_$v.so python tools/prof_sweep.py vehicle3d 2>&1 | tail -1)"
done
