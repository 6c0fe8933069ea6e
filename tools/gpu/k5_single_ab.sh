for v in d128 s128 s256 d128 s128 s256; do
  echo "$v $(IMP_LIB_PATH=_variants/libimpact_b200_$v.so python tools/time_synth.py room5d 100 2>&1 | tail -1)"
  echo "$v $(IMP_LIB_PATH=_variants/libimpact_b200_$v.so python tools/time_synth.py vehicle3d 2>&1 | tail -1)"
done
