#!/bin/bash
# schedule_lpt 0 / 1 / 2 / 3 at the parity and the production tolerance, shifted and replayed inputs
set -u
for tol in "" "--rtol 1e-6 --atol 1e-12"; do
 for ev in shift restore; do
  for c in cfg3 cfg5; do
   for m in 0 1 2 3; do
    timeout 600 python bench.py --config $c --steps 6 --warmup 2 --evolve $ev $tol --opt schedule_lpt=$m --also none --no-schedules --no-prod --no-e2e --no-cpu-baseline > gpurun_out/lm.json 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/lm.json').read().strip().splitlines()[-1]);print('tol=${tol:-parity} ev=$ev $c lpt_opt=$m', round(d['value'],1), 'ran', d['detail']['lpt'])"
   done
  done
 done
done
