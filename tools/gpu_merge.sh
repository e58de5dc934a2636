mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "merge" > gpurun_out/pytest_merge.txt 2>&1; tail -3 gpurun_out/pytest_merge.txt
timeout 900 python tools/merge_bench.py C1 C2 C3 C5_p0.001 C5_p0.01 | tee gpurun_out/merge_bench.jsonl
