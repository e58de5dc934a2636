set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
./tools/swar_ubench > gpurun_out/ubench.txt 2>&1; cat gpurun_out/ubench.txt
timeout 900 python -m pytest tests -m gpu -x -q -k "not c4 and not c3 and not c5" > gpurun_out/pytest_gpu1.txt 2>&1; tail -30 gpurun_out/pytest_gpu1.txt
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; cat gpurun_out/bench1.json; tail -20 gpurun_out/bench1.err
