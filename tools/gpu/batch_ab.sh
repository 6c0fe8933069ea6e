for b in 4 8 16 32; do
  echo "batch=$b $(IMPACT_REFINE_BATCH=$b python tools/time_build.py vehicle3d 2>&1 | tail -1)"
done
for b in 4 16; do
  echo "batch=$b $(IMPACT_REFINE_BATCH=$b python tools/time_build.py room5d once 2>&1 | tail -1)"
done
