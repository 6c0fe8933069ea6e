#!/bin/bash
# Time vehicle3d / room5d refine throughput under JIT tuning knobs.
rate() { python -c "import sys,re; s=sys.stdin.read(); m=re.search(r'ms_refine=([0-9.]+).*nm_evals=([0-9]+)', s); print('  evals/s %.3e' % (int(m.group(2))/float(m.group(1))*1e3) if m else s)"; }
for cfg in "vehicle3d 2500 100" "room5d 2500 60"; do
for minb in 2 4; do for ch in 0 1; do
  echo "$cfg minb=$minb chunk=$ch"
  IMPACT_REFINE_MINB=$minb IMPACT_NDTR_CHUNK=$ch timeout 120 python tools/prof_build.py $cfg 2>&1 | tail -1 | rate
done; done; done
