#!/bin/bash
set -u
mkdir -p gpurun_out
for c in cfg2 cfg5; do
  for k in 3 5 8 12; do
    timeout 900 python bench.py --config $c --steps 6 --warmup 2 --e2e-chunks $k --also none --no-schedules --no-prod --no-cpu-baseline > gpurun_out/e2e_${c}_$k.json 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/e2e_${c}_$k.json').read().strip().splitlines()[-1]);print('$c','$k',round(d['value'],1),round(d['e2e']['value'],1))"
  done
done
