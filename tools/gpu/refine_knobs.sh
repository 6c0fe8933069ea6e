# k_refine JIT knob sweep on the full vehicle3d build (fast objective)
for u in 0 1; do for c in 1 2 3; do for m in 4 5 6 8; do
  echo "unroll=$u chunk=$c minb=$m: $(IMPACT_NDTR_UNROLL=$u IMPACT_NDTR_CHUNK=$c IMPACT_REFINE_MINB=$m timeout 120 python tools/time_build.py vehicle3d once 2>&1 | tail -1)"
done; done; done
