#!/bin/bash
# NEXT-2 on the round-2 build: K_max_bulk x N* under Alg. 3 and the default (in-call heavy-first)
# schedule on cfg3/cfg4/cfg5, the paper's all-cells bulk mode, and the fusion crossover (App. E).
set -u
mkdir -p gpurun_out
timeout 2400 python tools/sweep_schedule.py cfg3 cfg4 cfg5 --kmax 1,5,20 --nstar 1e4,-1,3e5,1e9 --lpt 0,2 > gpurun_out/r02_next2_sweep.jsonl 2> gpurun_out/r02_next2_sweep.err
tail -3 gpurun_out/r02_next2_sweep.err
wc -l gpurun_out/r02_next2_sweep.jsonl
