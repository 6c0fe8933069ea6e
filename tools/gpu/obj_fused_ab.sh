for r in 1 2; do
for f in 0 1 2; do
  echo "fused=$f $(IMPACT_OBJ_FUSED=$f python tools/time_build.py vehicle3d 2>&1 | tail -1)"
done
done
for f in 0 1 2; do
  echo "fused=$f $(IMPACT_OBJ_FUSED=$f python tools/time_build.py room5d once 2>&1 | tail -1)"
done
