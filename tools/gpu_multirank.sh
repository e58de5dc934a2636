mkdir -p gpurun_out
export BENCH_DIST_BACKEND=gloo BENCH_FORCE_DEVICE=0
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench_2rank.json 2> gpurun_out/bench_2rank.err
echo "rc=$?"; cat gpurun_out/bench_2rank.json | cut -c1-600; tail -5 gpurun_out/bench_2rank.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/bench_ref2.json 2> gpurun_out/bench_ref2.err
echo "rc=$?"; cat gpurun_out/bench_ref2.json | cut -c1-400
