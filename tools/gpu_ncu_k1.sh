mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1_conc_small -s 2 -c 1 -o gpurun_out/k1_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_k1.log 2>&1; tail -2 gpurun_out/ncu_k1.log
