# K1 byte tier v2 (persistent lanes, IPC): tier tests, C5 sweep, build timings of both tiers with checks, launch lists.
mkdir -p gpurun_out
TAG=${TAG:-r2c}
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "tiers or invariants or sharded or colliding or randomized or c1_ or c2_ or c3_ or c4_ or c5_ or mixed or promoted or golden or bytes" > gpurun_out/pytest_k1_$TAG.txt 2>&1; tail -3 gpurun_out/pytest_k1_$TAG.txt
timeout 900 python -m pytest tests/test_gpu_c5_sweep.py -m gpu -q -x > gpurun_out/pytest_c5_$TAG.txt 2>&1; tail -2 gpurun_out/pytest_c5_$TAG.txt
timeout 1200 python tools/build_bench.py --check --variants "byte=1;byte=1,ipc=1;byte=0" C1 C2 C3 C4 C5_p0.001 C5_p0.01 C5_p0.05 C5_p0.1 > gpurun_out/build_bench_$TAG.jsonl 2> gpurun_out/build_bench_$TAG.err; cat gpurun_out/build_bench_$TAG.jsonl; tail -3 gpurun_out/build_bench_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/k1_launches_C4_$TAG.csv python tools/build_once.py C4 --n 2 > gpurun_out/k1_launches_C4_$TAG.log 2>&1; tail -1 gpurun_out/k1_launches_C4_$TAG.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1_byte -s 1 -c 1 -o gpurun_out/k1_byte_C5p10_$TAG python tools/build_once.py C5_p0.1 --n 2 > gpurun_out/ncu_k1_C5p10_$TAG.log 2>&1; tail -2 gpurun_out/ncu_k1_C5p10_$TAG.log
