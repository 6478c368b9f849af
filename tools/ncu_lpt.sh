#!/bin/bash
# per-launch metrics of the integration kernels on cfg3 (warm-up call: bulk-sparse; later calls: the
# heavy-first persistent lockstep launch)
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.per_cycle_active,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio,smsp__thread_inst_executed_per_inst_executed.ratio \
  --clock-control none -k regex:k_integrate --csv --log-file gpurun_out/${1:-r}_ncu_cfg3_lpt.csv \
  python bench.py --config cfg3 --steps 1 --warmup 2 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python - <<'PY'
import csv, collections, sys
rows = [r for r in csv.reader(open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/${1:-r}_ncu_cfg3_lpt.csv")) if len(r) > 10]
PY
