#!/bin/bash
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/h0_smi.txt
for c in cfg2 cfg5 cfg3; do
 for h in 0.01 0.03 0.1 0.3 1.0; do
  echo -n "$c h0=$h " >> gpurun_out/h0_sweep.txt
  timeout 300 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --h0 $h 2>>gpurun_out/h0_err.txt | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2), 'frac', round(d['roofline']['frac'],3), 'ms', round(d['ms_per_step'],2), 'sub', round(d['detail']['substeps_per_cell_step'],3))" >> gpurun_out/h0_sweep.txt 2>&1
 done
done
cat gpurun_out/h0_sweep.txt
