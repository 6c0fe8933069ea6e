for v in walkf0 walkf2 walkf1; do
  for c in robot2d_reachavoid vehicle3d; do
    echo "$v $(IMP_LIB_PATH=_variants/libimpact_b200_$v.so python tools/time_synth.py $c 2>&1 | tail -1)"
  done
  echo "$v $(IMP_LIB_PATH=_variants/libimpact_b200_$v.so python tools/time_synth.py room5d 100 2>&1 | tail -1)"
done
IMP_SWEEP_STATS=1 IMP_LIB_PATH=_variants/libimpact_b200_walkf2.so python tools/time_synth.py room5d 100 2>&1 | grep "imp\]" | head -1
