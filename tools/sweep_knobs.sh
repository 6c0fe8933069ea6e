#!/bin/bash
# Time k_refine throughput (evals/s) under JIT tuning knobs on config subsets.
rate() { python -c "import sys,re; s=sys.stdin.read(); m=re.search(r'ms_refine=([0-9.]+).*nm_evals=([0-9]+)', s); print('  evals/s %.3e' % (int(m.group(2))/float(m.group(1))*1e3) if m else s[-300:])"; }
for cfg in "vehicle3d 2500 600" "room5d 2500 200"; do
for minb in ${MINBS:-4 6}; do for ch in ${CHUNKS:-1}; do for vote in ${VOTES:-0 1}; do
  echo "$cfg minb=$minb chunk=$ch vote=$vote"
  IMPACT_NDTR_VOTE=$vote IMPACT_REFINE_MINB=$minb IMPACT_NDTR_CHUNK=$ch timeout 120 python tools/prof_build.py $cfg 2>&1 | tail -1 | rate
done; done; done; done
