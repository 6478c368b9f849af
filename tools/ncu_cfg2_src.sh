#!/bin/bash
# one --set full capture (with source) of the cfg2 bulk k_integrate launch, report kept in gpurun_out/
mkdir -p gpurun_out
TAG=${1:-src}
ncu --set full --clock-control none --import-source on -k regex:k_integrate -c 1 -f -o gpurun_out/${TAG}_cfg2 \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS:-} > gpurun_out/${TAG}_ncu.log 2>&1
ls -la gpurun_out/
