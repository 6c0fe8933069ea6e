for v in pf cur; do
  for c in robot2d_reachavoid robot2d_reach; do
    echo "$v $(IMP_LIB_PATH=_variants/libimpact_b200_$v.so python tools/time_synth.py $c 2>&1 | tail -1)"
  done
  echo "$v $(IMP_LIB_PATH=_variants/libimpact_b200_$v.so python tools/prof_sweep.py robot2d_reachavoid 2>&1 | tail -1)"
  echo "$v $(IMP_LIB_PATH=_variants/libimpact_b200_$v.so python tools/time_synth.py room5d 100 2>&1 | tail -1)"
done
IMP_LIB_PATH=_variants/libimpact_b200_pf.so python -m pytest tests/test_synthesis_gpu.py tests/test_fullsize_parity_gpu.py -m gpu -q -x -k "robot2d or random or shard" > gpurun_out/t18.log 2>&1
