# ncu --set full of in-loop K5 launches (phase loop of a benchmark config)
# Usage: tools/gpu/ncu_k5_inloop.sh TAG CFG SKIP COUNT [horizon]
TAG=$1; CFG=$2; SKIP=$3; CNT=$4; HOR=$5
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_sweep -s $SKIP -c $CNT \
  -o gpurun_out/k5_$TAG python tools/prof_phase.py $CFG $HOR > gpurun_out/ncu_k5_$TAG.log 2>&1
python tools/ncu_summary.py gpurun_out/k5_$TAG.ncu-rep > gpurun_out/ncu_k5_$TAG.txt 2>&1
