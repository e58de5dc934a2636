# Several ranks on one GPU over gloo (test hook): distributed exactness check, then the bench at N=2, 3
mkdir -p gpurun_out
export BENCH_DIST_BACKEND=gloo BENCH_FORCE_DEVICE=0
for N in 2 3; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2954$N tools/dist_check.py C1 C3 > gpurun_out/dist_check_$N.txt 2>&1
echo "dist_check N=$N rc=$?"; grep exact gpurun_out/dist_check_$N.txt
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench_2rank.json 2> gpurun_out/bench_2rank.err
echo "rc=$?"; cat gpurun_out/bench_2rank.json | cut -c1-600; tail -5 gpurun_out/bench_2rank.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/bench_ref2.json 2> gpurun_out/bench_ref2.err
echo "rc=$?"; cat gpurun_out/bench_ref2.json | cut -c1-400
