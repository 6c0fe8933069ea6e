for c in "" 0 50 65 75 100; do
  echo "carveout=$c $(env ${c:+IMPACT_REFINE_CARVEOUT=$c} python tools/time_build.py vehicle3d 2>&1 | tail -1)"
done
echo "carveout= $(python tools/time_build.py room5d once 2>&1 | tail -1)"
echo "carveout=0 $(IMPACT_REFINE_CARVEOUT=0 python tools/time_build.py room5d once 2>&1 | tail -1)"
