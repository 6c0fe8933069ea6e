for v in cur e256 e512 cur e256 e512; do
  echo "$v $(IMP_LIB_PATH=_variants/libimpact_b200_$v.so python tools/time_synth.py vehicle3d 2>&1 | tail -1)"
  echo "$v $(IMP_LIB_PATH=_variants/libimpact_b200_$v.so python tools/time_synth.py dim14_verify 100 2>&1 | tail -1)"
done
