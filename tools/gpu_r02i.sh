#!/bin/bash
# r02i: RODAS3 vs RODAS4 (parity and production tolerance), 2-rank gloo runs of the N>1 path on one GPU
# (cfg4 LPT plan + per-step reductions, cfg5 plan), compute-sanitizer over the schedule variants.
set -u
TAG=${1:-r02i}
mkdir -p gpurun_out
for m in rodas3 rodas4; do
  for c in cfg2 cfg3; do
    timeout 600 python bench.py --config $c --method $m --steps 10 --warmup 3 --also none --no-schedules --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_${m}_$c.json 2> gpurun_out/${TAG}_${m}_$c.err
    python tools/summarize_line.py gpurun_out/${TAG}_${m}_$c.json
  done
done
for c in cfg4 cfg5; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 \
     bench.py --gpus 2 --config $c --steps 3 --warmup 2 --backend gloo --no-schedules --no-prod --no-e2e > gpurun_out/${TAG}_2ranks_gloo_$c.json 2> gpurun_out/${TAG}_2ranks_gloo_$c.err
  tail -2 gpurun_out/${TAG}_2ranks_gloo_$c.err; python tools/summarize_line.py gpurun_out/${TAG}_2ranks_gloo_$c.json
  python -c "import json;d=json.loads(open('gpurun_out/${TAG}_2ranks_gloo_$c.json').read().strip().splitlines()[-1]);c=d['config'];print({k:c.get(k) for k in ('imbalance_max_over_mean','imbalance_without_lpt','boxes_owned','multi_gpu_status')}, d['detail']['step_reductions'])"
done
bash tools/sanitize.sh > gpurun_out/${TAG}_sanitize.txt 2>&1; cat gpurun_out/${TAG}_sanitize.txt
