#!/bin/bash
set -u
run() {
for tol in "" "--rtol 1e-6 --atol 1e-12"; do
  for c in cfg2 cfg2b cfg3 cfg4 cfg5; do
    timeout 600 python bench.py --config $c --steps 6 --warmup 2 $tol --opt lockstep=0 --also none --no-schedules --no-prod --no-e2e --no-cpu-baseline > gpurun_out/pa.json 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/pa.json').read().strip().splitlines()[-1]);print('$1 lock0 tol=${tol:-parity} $c', round(d['value'],1), 'lpt', d['detail']['lpt'], 'simt', round(d['detail']['bulk_simt_eff'],3))"
  done
done
}
run A
CHEM_NVCC_EXTRA="-DCHEM_BULK_PERSIST=1" python -m paper_2510_23993_b200.build --force > /dev/null 2>&1
run P1
