#!/bin/bash
# ncu evidence for profiles/: launch list of the default bench command, full captures of the cfg2
# bulk launch and of a cfg5 lockstep burst.  Reports stay in /tmp (too big for gpurun_out); summaries
# are printed into gpurun_out/.
set -u
TAG=${1:-r1e}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_cfg2.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_integrate -c 1 -f -o /tmp/${TAG}_cfg2 \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_integrate --launch-skip 1 -c 1 -f -o /tmp/${TAG}_cfg5lock \
    python bench.py --config cfg5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --opt lockstep=1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio,smsp__thread_inst_executed_per_inst_executed.ratio,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__block_size \
    --clock-control none -k regex:k_integrate -c 4 --csv --log-file gpurun_out/${TAG}_cfg5_nolock_metrics.csv \
    python bench.py --config cfg5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --opt lockstep=0 > /dev/null 2>&1
python tools/ncu_summary.py /tmp/${TAG}_cfg2.ncu-rep > gpurun_out/${TAG}_ncu_cfg2.txt
python tools/ncu_summary.py /tmp/${TAG}_cfg5lock.ncu-rep > gpurun_out/${TAG}_ncu_cfg5lock.txt
cat gpurun_out/${TAG}_ncu_cfg2.txt gpurun_out/${TAG}_ncu_cfg5lock.txt | grep -E "==|duration|no_instruction|wait_per|fp64|dram|warps_active|grid"
