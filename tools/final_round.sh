#!/bin/bash
# Round-end evidence in one gpurun call: GPU tests, smoke, full bench lines (cpu_baseline + e2e) of
# every config, the reference (oracle) arm, the ncu launch list of the default bench command and
# --set full captures of the cfg2 bulk launch and of a cfg5 lockstep burst (summaries in gpurun_out/).
set -u
TAG=${1:-final}
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > gpurun_out/${TAG}_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1
for c in cfg2 cfg3 cfg4 cfg5; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err
done
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/${TAG}_bench_reference.json 2> gpurun_out/${TAG}_bench_reference.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_cfg2.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_integrate -c 1 -f -o /tmp/${TAG}_cfg2 \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_integrate --launch-skip 1 -c 1 -f -o /tmp/${TAG}_cfg5lock \
    python bench.py --config cfg5 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --opt lockstep=1 > /dev/null 2>&1
python tools/ncu_summary.py /tmp/${TAG}_cfg2.ncu-rep > gpurun_out/${TAG}_ncu_cfg2.txt
python tools/ncu_summary.py /tmp/${TAG}_cfg5lock.ncu-rep > gpurun_out/${TAG}_ncu_cfg5lock.txt
cp /tmp/${TAG}_cfg2.ncu-rep gpurun_out/ 2>/dev/null
cat gpurun_out/${TAG}_tests.txt gpurun_out/${TAG}_smoke.txt | tail -4
for c in cfg2 cfg3 cfg4 cfg5 reference; do tail -c 400 gpurun_out/${TAG}_bench_$c.json; echo; done
