#!/bin/bash
# quick bench of the given configs (default all); prints one summary line per config
for c in ${CONFIGS:-cfg2 cfg3 cfg4 cfg5}; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 2 --no-cpu-baseline --no-e2e $QB_ARGS 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['value'],2), 'frac', round(d['roofline']['frac'],3), 'ms', round(d['ms_per_step'],2))"
done
