#!/bin/bash
# On the GPU box: measured DFMA peak (CUDA events) and the dynamic FP64 op count of libdevice exp/log
# (ncu).  Writes gpurun_out/fp64_peak.json and gpurun_out/fp64_ops.csv.
set -u
mkdir -p gpurun_out
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/fp64_probe tools/probes/fp64_probe.cu
/tmp/fp64_probe 4000 > gpurun_out/fp64_peak.json
ncu --clock-control none -k regex:'k_exp|k_log' --metrics \
  sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active \
  --csv /tmp/fp64_probe 10 > gpurun_out/fp64_ops.csv 2>&1
ncu --clock-control none -k regex:dfma_peak -c 1 --metrics sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg.per_second,gpu__time_duration.sum \
  --csv /tmp/fp64_probe 400 > gpurun_out/fp64_peak_ncu.csv 2>&1
cat gpurun_out/fp64_peak.json
