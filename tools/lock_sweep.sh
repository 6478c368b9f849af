for c in cfg2 cfg3 cfg4; do for o in "" "--opt lockstep=1"; do
 echo -n "$c [$o] "; timeout 300 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --no-e2e $o 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2), 'ms', round(d['ms_per_step'],2), 'lock', d['detail']['lockstep'])"
done; done
