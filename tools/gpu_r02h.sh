#!/bin/bash
# r02h: GRI (NEXT-3) bench lines at parity and production tolerance, DRAM traffic of k_integrate per
# config, ncu --set full of the cfg2 launch, and the launch list of the default bench command.
set -u
TAG=${1:-r02h}
mkdir -p gpurun_out
for c in cfg2 cfg3; do
  for tol in "" "--rtol 1e-6 --atol 1e-12"; do
    nm=$([ -z "$tol" ] && echo parity || echo prod)
    timeout 900 python bench.py --mech gri30_hon --config $c --steps 3 --warmup 2 --also none --no-prod --no-e2e --no-schedules $tol > gpurun_out/${TAG}_gri_${c}_$nm.json 2> gpurun_out/${TAG}_gri_${c}_$nm.err
    python tools/summarize_line.py gpurun_out/${TAG}_gri_${c}_$nm.json; tail -1 gpurun_out/${TAG}_gri_${c}_$nm.err
  done
done
for c in cfg2 cfg3 cfg4 cfg5; do
  ncu --clock-control none -k regex:k_integrate --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv \
     python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --also none --no-schedules --no-prod > gpurun_out/${TAG}_traffic_$c.csv 2>/dev/null
done
python tools/traffic.py $TAG cfg2 cfg3 cfg4 cfg5
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_cfg2.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --also none --no-schedules --no-prod > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_integrate -c 1 -f -o gpurun_out/${TAG}_cfg2 \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --also none --no-schedules --no-prod > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/${TAG}_cfg2.ncu-rep > gpurun_out/${TAG}_ncu_cfg2.txt 2>&1
head -12 gpurun_out/${TAG}_ncu_cfg2.txt
