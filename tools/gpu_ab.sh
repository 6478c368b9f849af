#!/bin/bash
# A/B of kernel build variants on one box: A = the shipped build; each further arg is a CHEM_NVCC_EXTRA
# flag set (quoted) rebuilt on the box and benched the same way.  Usage: gpu_ab.sh TAG "-DX" "-DY -DZ"
set -u
TAG=$1; shift
mkdir -p gpurun_out
run() {
  for c in ${CONFIGS:-cfg2 cfg3}; do
    timeout 600 python bench.py --config $c --steps 10 --warmup 3 --also none --no-schedules --no-prod --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_$1_$c.json 2> gpurun_out/${TAG}_$1_$c.err
    python tools/summarize_line.py gpurun_out/${TAG}_$1_$c.json | head -1
  done
}
echo "== A (shipped)"; run A
i=0
for flags in "$@"; do
  i=$((i+1))
  CHEM_NVCC_EXTRA="$flags" python -m paper_2510_23993_b200.build --force > /dev/null 2>&1 || { echo "build $flags failed"; continue; }
  grep -A2 "k_integrateI17Mech_h2air_li2004NS_6Rodas4ELi32ELb0" paper_2510_23993_b200/build.log | grep -E "spill" | head -1
  echo "== V$i ($flags)"; run V$i
done
