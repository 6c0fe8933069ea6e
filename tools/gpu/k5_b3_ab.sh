for v in b0 b2 b3 b0 b2 b3; do
  echo "$v $(IMP_LIB_PATH=_variants/libimpact_b200_$v.so python tools/time_synth.py room5d 100 2>&1 | tail -1)"
done
for v in b0 b2 b3; do
  echo "$v $(IMP_LIB_PATH=_variants/libimpact_b200_$v.so python tools/prof_sweep.py room5d 2>&1 | tail -1)"
  echo "$v $(IMP_LIB_PATH=_variants/libimpact_b200_$v.so python tools/time_synth.py vehicle3d 2>&1 | tail -1)"
done
IMP_SWEEP_STATS=1 IMP_LIB_PATH=_variants/libimpact_b200_b0.so python tools/time_synth.py room5d 100 2>&1 | grep "imp\]" | head -1
IMP_SWEEP_STATS=1 IMP_LIB_PATH=_variants/libimpact_b200_b3.so python tools/time_synth.py room5d 100 2>&1 | grep "imp\]" | head -1
