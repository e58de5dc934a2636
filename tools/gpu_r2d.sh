# K1 policy + async K2 host plan + cost-dealt sharded build: parity, build timings, part balance.
mkdir -p gpurun_out
TAG=${TAG:-r2d}
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c5_sweep.py tests/test_gpu_dist.py -m gpu -q -x > gpurun_out/pytest_$TAG.txt 2>&1; tail -3 gpurun_out/pytest_$TAG.txt
timeout 1200 python tools/build_bench.py --check --variants "byte=1;byte=0;byte=all" C1 C2 C3 C4 C5_p0.001 C5_p0.01 C5_p0.05 C5_p0.1 > gpurun_out/build_bench_$TAG.jsonl 2> gpurun_out/build_bench_$TAG.err; cat gpurun_out/build_bench_$TAG.jsonl | cut -c1-400; tail -3 gpurun_out/build_bench_$TAG.err
timeout 1500 python tools/part_balance.py C4 C5_p0.01 C2 C5_p0.1 > gpurun_out/part_balance_$TAG.jsonl 2> gpurun_out/part_balance_$TAG.err; tail -3 gpurun_out/part_balance_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/k1_launches_C4_$TAG.csv python tools/build_once.py C4 --n 2 > gpurun_out/k1_launches_C4_$TAG.log 2>&1; tail -1 gpurun_out/k1_launches_C4_$TAG.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1_byte -c 1 -o gpurun_out/k1_byte_C4_$TAG python tools/build_once.py C4 --n 1 > gpurun_out/ncu_k1_C4_$TAG.log 2>&1; tail -1 gpurun_out/ncu_k1_C4_$TAG.log
