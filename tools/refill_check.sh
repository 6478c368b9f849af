#!/bin/bash
# sparse-launch refill batch by list order: default schedule, Alg. 3 and sparse-only (N* = 1e9) per config
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/rf_tests.txt 2>&1; tail -1 gpurun_out/rf_tests.txt
for c in cfg2 cfg2b cfg3 cfg4 cfg5; do
  for o in "" "--opt schedule_lpt=0" "--opt n_active_star=1000000000"; do
    timeout 600 python bench.py --config $c --steps 5 --warmup 3 --also none --no-schedules --no-prod --no-e2e --no-cpu-baseline $o > gpurun_out/rf.json 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/rf.json').read().strip().splitlines()[-1]);print('$c [$o]', round(d['value'],1), 'lpt', d['detail']['lpt'], 'launches', d['gpu_launches'])"
  done
done
