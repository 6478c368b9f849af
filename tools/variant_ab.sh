#!/bin/bash
# A/B of prebuilt libchem variants (variants/libchem_<tag>.so, built here with CHEM_NVCC_EXTRA=...):
# kernel-only bench lines per config.  Usage: VARIANTS="bs32 bs64" CONFIGS="cfg2 cfg3" bash tools/variant_ab.sh TAG
set -u
TAG=${1:-v}
mkdir -p gpurun_out
cp paper_2510_23993_b200/libchem.so /tmp/libchem_default.so
for v in ${VARIANTS}; do
  cp variants/libchem_$v.so paper_2510_23993_b200/libchem.so
  for c in ${CONFIGS:-cfg2 cfg2b cfg3 cfg5}; do
    timeout 600 python bench.py --config $c --steps 6 --warmup 3 --also none --no-schedules --no-prod --no-e2e --no-cpu-baseline ${BENCH_ARGS:-} > gpurun_out/${TAG}_${v}_${c}.json 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/${TAG}_${v}_${c}.json').read().strip().splitlines()[-1]);print('$v $c', round(d['value'],1), 'frac', round(d['roofline']['frac'],3), 'lpt', d['detail']['lpt'])" 2>&1 | tail -1
  done
done
cp /tmp/libchem_default.so paper_2510_23993_b200/libchem.so
