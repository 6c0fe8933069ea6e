#!/bin/bash
# Lightweight ncu (few sections) of one kernel.  Usage: tools/ncu_quick.sh TAG KREGEX cmd...
TAG=$1; K=$2; shift 2
"$@" > gpurun_out/plain_q_$TAG.log 2>&1 && \
timeout 500 ncu --section SpeedOfLight --section WarpStateStats --section SchedulerStats \
  --section ComputeWorkloadAnalysis --section Occupancy --section LaunchStats --section InstructionStats \
  --metrics sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed_pipe_fp64.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum \
  --clock-control none -k regex:$K -s ${KSKIP:-0} -c 1 -o gpurun_out/q_$TAG "$@" > gpurun_out/ncu_q_$TAG.log 2>&1
tail -1 gpurun_out/ncu_q_$TAG.log
