for m in 5 4 6; do
  echo "minb=$m $(IMPACT_REFINE_MINB=$m python tools/time_build.py vehicle3d 2>&1 | tail -1)"
done
for m in 4 3; do
  echo "minb=$m $(IMPACT_REFINE_MINB=$m python tools/time_build.py room5d once 2>&1 | tail -1)"
done
