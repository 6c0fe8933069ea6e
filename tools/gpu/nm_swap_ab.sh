for r in 1 2; do
echo "head $(IMP_LIB_PATH=_variants/libimpact_b200_nmhead.so python tools/time_build.py vehicle3d 2>&1 | tail -1)"
echo "new0 $(IMPACT_NM_SWAP=0 IMP_LIB_PATH=_variants/libimpact_b200_nmswap.so python tools/time_build.py vehicle3d 2>&1 | tail -1)"
echo "new1 $(IMPACT_NM_SWAP=1 IMP_LIB_PATH=_variants/libimpact_b200_nmswap.so python tools/time_build.py vehicle3d 2>&1 | tail -1)"
done
echo "head $(IMP_LIB_PATH=_variants/libimpact_b200_nmhead.so python tools/time_build.py room5d once 2>&1 | tail -1)"
echo "new0 $(IMPACT_NM_SWAP=0 IMP_LIB_PATH=_variants/libimpact_b200_nmswap.so python tools/time_build.py room5d once 2>&1 | tail -1)"
echo "new1 $(IMPACT_NM_SWAP=1 IMP_LIB_PATH=_variants/libimpact_b200_nmswap.so python tools/time_build.py room5d once 2>&1 | tail -1)"
