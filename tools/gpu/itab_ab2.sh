for v in head new; do
echo "$v: $(IMP_LIB_PATH=_variants/libimpact_b200_$v.so python tools/time_build.py vehicle3d 2>&1 | tail -1)"
echo "$v notab: $(IMPACT_NO_INIT_TABLE=1 IMP_LIB_PATH=_variants/libimpact_b200_$v.so python tools/time_build.py vehicle3d 2>&1 | tail -1)"
done
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv
