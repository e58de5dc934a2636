mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_merge -c 1 -o gpurun_out/merge_full python tools/merge_bench.py C2 > gpurun_out/ncu_merge.log 2>&1; tail -2 gpurun_out/ncu_merge.log
