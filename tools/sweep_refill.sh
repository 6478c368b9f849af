#!/bin/bash
# default schedule vs lane-refill bulk bursts vs sparse-only (one persistent refill launch) per config
mkdir -p gpurun_out
for c in cfg2 cfg3 cfg4 cfg5; do
 for o in "" "--opt refill_bulk=1" "--opt n_active_star=1000000000000"; do
   echo -n "$c [$o] " >> gpurun_out/refill_sweep.txt
   timeout 300 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --no-e2e $o 2>>gpurun_out/refill_err.txt | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2), 'ms', round(d['ms_per_step'],2), 'launches', d['detail']['integrate_launches'], 'simt', round(d['detail'].get('bulk_simt_eff') or 0,3))" >> gpurun_out/refill_sweep.txt 2>&1
 done
done
cat gpurun_out/refill_sweep.txt
