#!/bin/bash
# Round-2 evidence in one gpurun call.  Output: gpurun_out/final_* (copied to profiles/ afterwards).
set -u
T=${T:-final}
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -s --durations=8 > gpurun_out/${T}_tests_full.txt 2>&1
grep -E "passed|failed|self-convergence|gap at" gpurun_out/${T}_tests_full.txt | tail -8
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.txt 2>&1; cat gpurun_out/${T}_smoke.txt
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/${T}_bench_cfg2.json 2> gpurun_out/${T}_bench_cfg2.err
for c in cfg3 cfg4 cfg5; do
  timeout 1200 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/${T}_bench_$c.json 2> gpurun_out/${T}_bench_$c.err
done
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/${T}_bench_reference.json 2> gpurun_out/${T}_bench_reference.err
for c in cfg2 cfg3 cfg4 cfg5; do tail -1 gpurun_out/${T}_bench_$c.err; python tools/summarize_line.py gpurun_out/${T}_bench_$c.json; done
tail -c 300 gpurun_out/${T}_bench_reference.json; echo
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_cfg2.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --also none --no-prod > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_cfg3.csv \
    python bench.py --config cfg3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-schedules --no-prod > /dev/null 2>&1
for c in cfg2 cfg3 cfg4 cfg5; do
  ncu --clock-control none -k regex:k_integrate --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv \
     python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --also none --no-schedules --no-prod > gpurun_out/${T}_traffic_$c.csv 2>/dev/null
done
ncu --set full --clock-control none --import-source on -k regex:k_integrate -c 1 -f -o gpurun_out/${T}_cfg2 \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --also none --no-schedules --no-prod > /dev/null 2>&1
# the timed call's two k_integrate launches (first lockstep burst + heavy-first persistent launch) after 3 warm-up
# calls (launches per call: 2, 1 on the cross-call hints of the second call, 2, 2)
ncu --set full --clock-control none --import-source on -k regex:k_integrate --launch-skip 5 -c 2 -f -o gpurun_out/${T}_cfg3lpt \
    python bench.py --config cfg3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --also none --no-schedules --no-prod > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/${T}_cfg2.ncu-rep > gpurun_out/${T}_ncu_cfg2.txt 2>&1
python tools/ncu_summary.py gpurun_out/${T}_cfg3lpt.ncu-rep > gpurun_out/${T}_ncu_cfg3lpt.txt 2>&1
head -14 gpurun_out/${T}_ncu_cfg2.txt; head -6 gpurun_out/${T}_ncu_cfg3lpt.txt
