# Round 2 (x): balanced mode for accumulated K2 items -- parity (full GPU suite), A/B timings, stress, ncu C3.
mkdir -p gpurun_out
TAG=${TAG:-r2x}
for b in 1 0 1 0; do for cfg in C3 C1; do BATMAP_K2_BALANCE=$b timeout 120 python tools/run_one.py $cfg 9 >> gpurun_out/bal_$TAG.txt 2>&1; echo "balance=$b" >> gpurun_out/bal_$TAG.txt; done; done; cat gpurun_out/bal_$TAG.txt
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$TAG.txt 2>&1; tail -2 gpurun_out/pytest_gpu_$TAG.txt
STRESS_SEED=99 timeout 500 python tools/stress.py 360 > gpurun_out/stress_$TAG.txt 2>&1; tail -1 gpurun_out/stress_$TAG.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k2_tiled -s 2 -c 1 -o gpurun_out/k2_C3_$TAG python tools/run_one.py C3 3 > gpurun_out/ncu_k2c3_$TAG.log 2>&1; tail -1 gpurun_out/ncu_k2c3_$TAG.log
timeout 900 python tools/run_configs.py C1 C2 C3 C4 > gpurun_out/configs_$TAG.jsonl 2> gpurun_out/configs_$TAG.err; tail -2 gpurun_out/configs_$TAG.err
