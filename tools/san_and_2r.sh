bash tools/sanitize.sh
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --steps 3 --warmup 3 --backend gloo --no-cpu-baseline > gpurun_out/r1h_bench_cfg2_2ranks_gloo_1gpu.json 2> gpurun_out/r1h_2r_cfg2.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29532 bench.py --gpus 2 --config cfg4 --steps 2 --warmup 3 --backend gloo --no-cpu-baseline > gpurun_out/r1h_bench_cfg4_2ranks_gloo_1gpu.json 2> gpurun_out/r1h_2r_cfg4.err
tail -c 300 gpurun_out/r1h_bench_cfg2_2ranks_gloo_1gpu.json; echo; tail -c 300 gpurun_out/r1h_bench_cfg4_2ranks_gloo_1gpu.json
