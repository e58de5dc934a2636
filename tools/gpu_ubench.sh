mkdir -p gpurun_out
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv,noheader -lms 50 > gpurun_out/ubench_clocks.csv &
SMI=$!
./tools/swar_ubench | tee gpurun_out/ubench4.txt
kill $SMI
timeout 300 ncu --metrics sm__cycles_elapsed.avg.per_second,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio,smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio,smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio --clock-control none ./tools/swar_ubench > gpurun_out/ubench4_ncu.txt 2>&1
