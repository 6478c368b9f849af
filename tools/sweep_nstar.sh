#!/bin/bash
# N* (bulk -> sparse switch) x K_max sweep on the tail-heavy configs; one line per point in gpurun_out/
mkdir -p gpurun_out
for c in cfg4 cfg3; do
 for ns in 10000 20000 37888 75000; do
  for km in 5 10; do
   echo -n "$c nstar=$ns kmax=$km " >> gpurun_out/nstar_sweep.txt
   timeout 300 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --opt n_active_star=$ns --opt kmax_bulk=$km 2>>gpurun_out/nstar_err.txt | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2), 'ms', round(d['ms_per_step'],2), 'launches', d['detail']['integrate_launches'])" >> gpurun_out/nstar_sweep.txt 2>&1
  done
 done
done
cat gpurun_out/nstar_sweep.txt
