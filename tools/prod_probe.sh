#!/bin/bash
set -u
for c in cfg5 cfg3; do
timeout 600 python bench.py --config $c --steps 6 --warmup 2 --rtol 1e-6 --atol 1e-12 --also none --no-schedules --no-prod --no-e2e --no-cpu-baseline > gpurun_out/prod_$c.json 2>/dev/null
python -c "
import json;d=json.loads(open('gpurun_out/prod_$c.json').read().strip().splitlines()[-1]);dd=d['detail']
print('$c', '${TAG:-A}', round(d['value'],1), {k:dd[k] for k in ('lpt','bulk_iters','sparse_cells','t_sparse_ms','k_integrate_ms','substeps_per_cell_step','active0')})"
done
