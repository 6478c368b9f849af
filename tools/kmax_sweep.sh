#!/bin/bash
# K_max of the bulk bursts (with it: the first burst before the in-call prediction) on the default schedule
set -u
mkdir -p gpurun_out
for km in 1 2 3 5 8; do
  for c in cfg2 cfg2b cfg3 cfg4 cfg5; do
    timeout 600 python bench.py --config $c --steps 8 --warmup 2 --also none --no-schedules --no-prod --no-e2e --no-cpu-baseline --opt kmax_bulk=$km > gpurun_out/km${km}_$c.json 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/km${km}_$c.json').read().strip().splitlines()[-1]);print('kmax $km $c', round(d['value'],1), round(d['roofline']['frac'],3), d['detail']['lpt'])"
  done
done
