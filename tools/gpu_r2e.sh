# NEXT-4 first GPU run + build-time fixes (pinned plan upload, mempool) check.
mkdir -p gpurun_out
TAG=${TAG:-r2e}
timeout 1200 python -m pytest tests/test_gpu_triples.py -m gpu -q -x --durations=10 > gpurun_out/pytest_triples_$TAG.txt 2>&1; tail -30 gpurun_out/pytest_triples_$TAG.txt
timeout 900 python tools/build_bench.py --check --variants "byte=1" C2 C3 C4 C5_p0.01 C5_p0.1 > gpurun_out/build_bench_$TAG.jsonl 2> gpurun_out/build_bench_$TAG.err; cat gpurun_out/build_bench_$TAG.jsonl | cut -c1-300; tail -3 gpurun_out/build_bench_$TAG.err
timeout 900 python tools/part_balance.py C4 --parts 8 > gpurun_out/part_balance_$TAG.jsonl 2> gpurun_out/part_balance_$TAG.err; tail -c 800 gpurun_out/part_balance_$TAG.jsonl
