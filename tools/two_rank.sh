#!/bin/bash
# the N>1 path on one GPU: 2 ranks over gloo (LPT box sharding, max-over-ranks timing)
mkdir -p gpurun_out
for c in cfg2 cfg4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2953${#c} \
    bench.py --gpus 2 --config $c --steps 3 --warmup 3 --backend gloo --no-cpu-baseline > gpurun_out/${1:-r}_bench_${c}_2ranks_gloo_1gpu.json 2> gpurun_out/${1:-r}_2r_$c.err
  tail -1 gpurun_out/${1:-r}_bench_${c}_2ranks_gloo_1gpu.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['n_gpus'], round(d['value'],1), d['config']['schedule'][:24], d['config'].get('imbalance_max_over_mean'))"
done
