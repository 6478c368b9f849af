for c in cfg4 cfg5; do for o in "" "--opt lockstep=0"; do
 echo -n "$c [$o] "; timeout 300 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --no-e2e $o 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2), 'ms', round(d['ms_per_step'],2), 'lock', d['detail']['lockstep'], 'simt', round(d['detail']['bulk_simt_eff'],3))"
done; done
