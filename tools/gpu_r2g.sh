# Full GPU suite, build trace with the new planner, bench (driver form), configs with K2 times.
mkdir -p gpurun_out
TAG=${TAG:-r2g}
BATMAP_TRACE=1 timeout 300 python tools/build_once.py C4 --n 3 > gpurun_out/trace_C4_$TAG.txt 2>&1; tail -9 gpurun_out/trace_C4_$TAG.txt
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$TAG.txt 2>&1; tail -2 gpurun_out/pytest_gpu_$TAG.txt
timeout 900 python tools/build_bench.py --check C2 C3 C4 C5_p0.01 C5_p0.1 > gpurun_out/build_bench_$TAG.jsonl 2> gpurun_out/build_bench_$TAG.err; cat gpurun_out/build_bench_$TAG.jsonl | cut -c1-250
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -c 1500 gpurun_out/bench_$TAG.json; tail -3 gpurun_out/bench_$TAG.err
