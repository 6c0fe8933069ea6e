# exact k_refine JIT knobs on the full vehicle3d / room5d builds
for u in 0 1; do for c in 1 2 3; do for m in 4 5; do
  echo "unroll=$u chunk=$c minb=$m: $(IMPACT_NDTR_UNROLL=$u IMPACT_NDTR_CHUNK=$c IMPACT_REFINE_MINB=$m timeout 120 python tools/time_build.py vehicle3d once 2>&1 | tail -1)"
done; done; done
for u in 0 1; do
  echo "room5d unroll=$u chunk=2 minb=5: $(IMPACT_NDTR_UNROLL=$u timeout 200 python tools/time_build.py room5d once 2>&1 | tail -1)"
done
