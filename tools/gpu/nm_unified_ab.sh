for u in 0 1 0 1; do
  echo "u=$u $(IMPACT_NM_UNIFIED=$u python tools/time_build.py vehicle3d 2>&1 | tail -1)"
done
for u in 0 1; do
  echo "u=$u $(IMPACT_NM_UNIFIED=$u python tools/time_build.py room5d once 2>&1 | tail -1)"
  echo "u=$u $(IMPACT_NM_UNIFIED=$u python tools/time_build.py bas7d_verify once 2>&1 | tail -1)"
done
