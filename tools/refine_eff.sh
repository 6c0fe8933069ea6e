#!/bin/bash
# k_refine SIMT efficiency (evals / lane slots) and throughput per config.
for a in "$@"; do
python tools/prof_build.py $a | python -c "
import sys,re; s=sys.stdin.read(); ev=int(re.search(r'nm_evals=(\d+)',s).group(1)); sl=int(re.search(r'nm_lane_slots=(\d+)',s).group(1)); ms=float(re.search(r'ms_refine=([0-9.]+)',s).group(1)); print('$a', 'eff %.3f' % (ev/sl if sl else 0), 'evals/s %.3e' % (ev/ms*1e3), 'refine ms %.1f' % ms)"
done
