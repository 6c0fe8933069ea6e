for v in old new t768 t512; do
  for c in robot2d_reachavoid vehicle3d; do
    echo "$v $(IMP_LIB_PATH=_variants/libimpact_b200_$v.so python tools/time_synth.py $c 2>&1 | tail -1)"
  done
  echo "$v $(IMP_LIB_PATH=_variants/libimpact_b200_$v.so python tools/time_synth.py dim14_verify 100 2>&1 | tail -1)"
done
