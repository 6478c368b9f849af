#!/bin/bash
# NEXT-3 evidence: GPU tests (incl. the 14-species mechanism), the DMMA probe (timed + ncu pipe
# utilisation per kernel), bench lines of the 14-species mechanism.
set -u
TAG=${1:-r02g}
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/${TAG}_tests.txt 2>&1
tail -3 gpurun_out/${TAG}_tests.txt
cd tools/probes && nvcc -O3 -std=c++17 --expt-relaxed-constexpr -gencode arch=compute_100a,code=sm_100a -o /tmp/dmma_probe dmma_probe.cu && cd ../..
/tmp/dmma_probe > gpurun_out/${TAG}_dmma.jsonl 2>&1
cat gpurun_out/${TAG}_dmma.jsonl
ncu --clock-control none --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.sum,smsp__inst_executed.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.per_cycle_active \
   --csv /tmp/dmma_probe > gpurun_out/${TAG}_dmma_ncu.csv 2>&1
grep -c "k_dmma" gpurun_out/${TAG}_dmma_ncu.csv
for c in cfg2 cfg3; do
  timeout 900 python bench.py --mech gri30_hon --config $c --steps 5 --warmup 3 --also none --no-prod --no-e2e > gpurun_out/${TAG}_bench_gri_$c.json 2> gpurun_out/${TAG}_bench_gri_$c.err
  tail -2 gpurun_out/${TAG}_bench_gri_$c.err; python tools/summarize_line.py gpurun_out/${TAG}_bench_gri_$c.json
done
