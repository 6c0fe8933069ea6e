python -m pytest tests/test_construct_gpu.py -m gpu -q -x -k "golden" > gpurun_out/t20.log 2>&1
for m in 5 6; do for c in 1 2; do
  echo "merge minb=$m chunk=$c: $(IMPACT_REFINE_MINB=$m IMPACT_NDTR_CHUNK=$c python tools/time_build.py vehicle3d once 2>&1 | tail -1)"
done; done
echo "room5d: $(IMPACT_NDTR_CHUNK=1 python tools/time_build.py room5d once 2>&1 | tail -1)"
echo "room5d chunk2: $(python tools/time_build.py room5d once 2>&1 | tail -1)"
