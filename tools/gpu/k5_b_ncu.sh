for v in b0 b2; do
IMP_LIB_PATH=_variants/libimpact_b200_$v.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_sweep -s 40 -c 30 --csv --log-file gpurun_out/k5t_$v.csv python tools/prof_phase.py room5d 30 > /dev/null 2>&1
done
