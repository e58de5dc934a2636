# Quick GPU check after a change: full GPU suite, selected configs, default bench.
mkdir -p gpurun_out
TAG=${TAG:-chk}
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$TAG.txt 2>&1; tail -3 gpurun_out/pytest_gpu_$TAG.txt
timeout 1200 python tools/run_configs.py ${CONFIGS:-C1 C2 C3} > gpurun_out/configs_$TAG.jsonl 2> gpurun_out/configs_$TAG.err; tail -3 gpurun_out/configs_$TAG.err
timeout 600 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -c 400 gpurun_out/bench_$TAG.json
