mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "not c4 and not c3" > gpurun_out/pytest_quick.txt 2>&1; tail -4 gpurun_out/pytest_quick.txt
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err; cat gpurun_out/bench_quick.json; tail -5 gpurun_out/bench_quick.err
