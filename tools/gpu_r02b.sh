#!/bin/bash
# r02b: GPU tests (with prints), smoke, fp64 probe, default bench line.
set -u
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -s -x --durations=15 > gpurun_out/r02b_tests_full.txt 2>&1
grep -E "self-convergence|gap at" gpurun_out/r02b_tests_full.txt > gpurun_out/r02b_conv.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02b_smoke.txt 2>&1
bash tools/fp64_probe.sh > /dev/null 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r02b_bench_cfg2.json 2> gpurun_out/r02b_bench_cfg2.err
tail -25 gpurun_out/r02b_tests_full.txt; cat gpurun_out/r02b_conv.txt gpurun_out/r02b_smoke.txt gpurun_out/fp64_peak.json
tail -c 1500 gpurun_out/r02b_bench_cfg2.json; tail -3 gpurun_out/r02b_bench_cfg2.err
