for v in ww32 ww64 ww32 ww64; do
  echo "$v $(IMP_LIB_PATH=_variants/libimpact_b200_$v.so python tools/time_synth.py room5d 100 2>&1 | tail -1)"
  echo "$v $(IMP_LIB_PATH=_variants/libimpact_b200_$v.so python tools/time_synth.py robot2d_reachavoid 2>&1 | tail -1)"
done
