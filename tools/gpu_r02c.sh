#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -s --durations=10 > gpurun_out/r02c_tests_full.txt 2>&1
grep -E "self-convergence|gap at" gpurun_out/r02c_tests_full.txt > gpurun_out/r02c_conv.txt
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r02c_bench_cfg2.json 2> gpurun_out/r02c_bench_cfg2.err
for c in cfg4 cfg5; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/r02c_bench_$c.json 2> gpurun_out/r02c_bench_$c.err
done
tail -15 gpurun_out/r02c_tests_full.txt; cat gpurun_out/r02c_conv.txt
for c in cfg2 cfg4 cfg5; do tail -3 gpurun_out/r02c_bench_$c.err; python tools/summarize_line.py gpurun_out/r02c_bench_$c.json; done
