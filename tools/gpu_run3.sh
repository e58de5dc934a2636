mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu3.txt 2>&1; tail -3 gpurun_out/pytest_gpu3.txt
timeout 1500 python tools/run_configs.py ${CONFIGS:-C1 C2 C3 C4 C5_p0.001 C5_p0.01 C5_p0.1} > gpurun_out/configs.jsonl 2> gpurun_out/configs.err; tail -3 gpurun_out/configs.err
