#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -s --durations=5 > gpurun_out/r02d_tests_full.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r02d_bench_cfg2.json 2> gpurun_out/r02d_bench_cfg2.err
for c in cfg4 cfg5; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02d_bench_$c.json 2> gpurun_out/r02d_bench_$c.err
done
ncu --set full --clock-control none --import-source on -k regex:k_integrate -c 1 -f -o gpurun_out/r02d_cfg2 \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --also none --no-schedules --no-prod > /dev/null 2>&1
tail -4 gpurun_out/r02d_tests_full.txt
for c in cfg2 cfg4 cfg5; do tail -2 gpurun_out/r02d_bench_$c.err; python tools/summarize_line.py gpurun_out/r02d_bench_$c.json; done
ls -la gpurun_out/r02d_cfg2.ncu-rep
