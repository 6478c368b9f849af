#!/bin/bash
# GPU tests + cfg2..cfg5 kernel-only bench lines with the schedule variants.  TAG as $1.
set -u
TAG=${1:-s}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${TAG}_tests.txt 2>&1
tail -2 gpurun_out/${TAG}_tests.txt
for c in ${CONFIGS:-cfg2 cfg3 cfg4 cfg5}; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --also none --no-prod --no-e2e --no-cpu-baseline ${BENCH_ARGS:-} > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err
  tail -1 gpurun_out/${TAG}_bench_$c.err; python tools/summarize_line.py gpurun_out/${TAG}_bench_$c.json
done
