mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "shard or tiers" > gpurun_out/pytest_shard.txt 2>&1; tail -3 gpurun_out/pytest_shard.txt
bash tools/gpu_multirank.sh
