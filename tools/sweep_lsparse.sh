#!/bin/bash
# sparse phase as free-running vs lockstep lane refill (chem_opts.lockstep_sparse), with the default
# N* and with sparse-only (N* huge)
for c in cfg3 cfg4 cfg5 cfg2; do
 for o in "" "--opt lockstep_sparse=1" "--opt lockstep_sparse=1 --opt n_active_star=1000000000000"; do
   echo -n "$c [$o] "
   timeout 300 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --no-e2e $o 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); dd=d['detail']; print(round(d['value'],2), 'ms', round(d['ms_per_step'],2), 'sparse_ms', round(dd['t_sparse_ms'],1), 'lock', dd['lockstep'])"
 done
done
