#!/bin/bash
# e2e copy/compute groups x taper (middle-group share / end-group share) for the pipelined fields
set -u
mkdir -p gpurun_out
for ch in 3 4 5; do for tp in 2 3 4; do
  python bench.py --config cfg2 --steps 10 --warmup 3 --also none --no-schedules --no-prod --no-cpu-baseline --e2e-chunks $ch --e2e-taper $tp > gpurun_out/tp.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/tp.json').read().strip().splitlines()[-1]);print('cfg2 chunks $ch taper $tp e2e', round(d['e2e']['value'],1), 'kernel', round(d['value'],1))"
done; done
for ch in 8 12 16; do for tp in 2 4; do
  python bench.py --config cfg5 --steps 4 --warmup 3 --also none --no-schedules --no-prod --no-cpu-baseline --e2e-chunks $ch --e2e-taper $tp > gpurun_out/tp.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/tp.json').read().strip().splitlines()[-1]);print('cfg5 chunks $ch taper $tp e2e', round(d['e2e']['value'],1), 'kernel', round(d['value'],1))"
done; done
