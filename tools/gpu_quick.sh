#!/bin/bash
# quick A/B: GPU tests + cfg2/cfg3 kernel-only bench lines.  TAG as $1.
set -u
TAG=${1:-q}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/${TAG}_tests.txt 2>&1
for c in ${CONFIGS:-cfg2 cfg3}; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --also none --no-schedules --no-prod --no-e2e --no-cpu-baseline ${BENCH_ARGS:-} > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err
done
tail -2 gpurun_out/${TAG}_tests.txt
for c in ${CONFIGS:-cfg2 cfg3}; do tail -2 gpurun_out/${TAG}_bench_$c.err; python tools/summarize_line.py gpurun_out/${TAG}_bench_$c.json; done
