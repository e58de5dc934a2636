# Round 2 (i): K2 block skipping + grouped tile order: GPU tests, configs, DRAM traffic of K2
# (default grouped order vs BATMAP_K2_GROUP=1 row-major) on C2 and C4.
mkdir -p gpurun_out
TAG=${TAG:-r2i}
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$TAG.txt 2>&1; tail -3 gpurun_out/pytest_gpu_$TAG.txt
timeout 1500 python tools/run_configs.py C1 C2 C3 C5_p0.001 C5_p0.01 > gpurun_out/configs_$TAG.jsonl 2> gpurun_out/configs_$TAG.err; tail -2 gpurun_out/configs_$TAG.err
BATMAP_K2_GROUP=1 timeout 900 python tools/run_configs.py C1 C2 C3 > gpurun_out/configs_${TAG}_g1.jsonl 2> gpurun_out/configs_${TAG}_g1.err; tail -2 gpurun_out/configs_${TAG}_g1.err
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct
for cfg in C2 C4; do
  timeout 900 ncu --metrics $M --clock-control none -k regex:k2_tiled -c 1 --csv python tools/run_one.py $cfg 1 > gpurun_out/k2_dram_${cfg}_$TAG.csv 2>&1
  BATMAP_K2_GROUP=1 timeout 900 ncu --metrics $M --clock-control none -k regex:k2_tiled -c 1 --csv python tools/run_one.py $cfg 1 > gpurun_out/k2_dram_${cfg}_${TAG}_g1.csv 2>&1
done
grep -h "dram__\|hit_rate\|gpu__time" gpurun_out/k2_dram_*_$TAG*.csv | cut -c1-220
