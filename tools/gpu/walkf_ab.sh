for v in walkf0 walkf1; do
  for c in robot2d_reachavoid robot2d_reach vehicle3d; do
    echo "$v $(IMP_LIB_PATH=_variants/libimpact_b200_$v.so python tools/time_synth.py $c 2>&1 | tail -1)"
  done
  echo "$v $(IMP_LIB_PATH=_variants/libimpact_b200_$v.so python tools/time_synth.py room5d 100 2>&1 | tail -1)"
done
IMP_LIB_PATH=_variants/libimpact_b200_walkf1.so python -m pytest tests/test_synthesis_gpu.py tests/test_fullsize_parity_gpu.py tests/test_sharded_gpu.py -m gpu -q -x -k "robot2d or random or shard or trace or golden_controller or wider" > gpurun_out/walkf_t.log 2>&1; tail -3 gpurun_out/walkf_t.log
