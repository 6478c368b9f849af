#!/bin/bash
# One gpurun call: GPU tests, smoke, bench lines for every config.  Output under gpurun_out/.
set -u
TAG=${1:-run}
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/${TAG}_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1
for c in ${CONFIGS:-cfg2 cfg3 cfg4 cfg5}; do
  timeout 900 python bench.py --config $c --steps ${STEPS:-10} --warmup 3 ${BENCH_ARGS:-} > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err
done
cat gpurun_out/${TAG}_tests.txt gpurun_out/${TAG}_smoke.txt | tail -8
for c in ${CONFIGS:-cfg2 cfg3 cfg4 cfg5}; do
  python - "$c" "gpurun_out/${TAG}_bench_$c.json" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    print(sys.argv[1], "value=%.2f" % d["value"], "frac=%.3f" % d["roofline"]["frac"], "e2e=%s" % (d["e2e"] or {}).get("value"),
          "cpu=%s" % (d["cpu_baseline"] or {}).get("value"), "substeps=%.2f" % d["detail"]["substeps_per_cell_step"],
          "act0=%d" % d["detail"]["active0"], "sparse=%d" % d["detail"]["sparse_cells"], "clk=%s" % d["clocks"].get("sm_mhz"))
except Exception as e:
    print(sys.argv[1], "FAILED", e)
PY
done
