# Round 2 (j): K2 block skipping (hoisted operand pointers) + grouped tile order: GPU tests, configs,
# K2 DRAM traffic vs the band height G (BATMAP_K2_GROUP) on C2 and C4.
mkdir -p gpurun_out
TAG=${TAG:-r2j}
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$TAG.txt 2>&1; tail -3 gpurun_out/pytest_gpu_$TAG.txt
timeout 1500 python tools/run_configs.py C1 C2 C3 C5_p0.001 > gpurun_out/configs_$TAG.jsonl 2> gpurun_out/configs_$TAG.err; tail -2 gpurun_out/configs_$TAG.err
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct
for G in 1 4 8 16 42; do
  BATMAP_K2_GROUP=$G timeout 300 ncu --metrics $M --clock-control none -k regex:k2_tiled -c 1 --csv python tools/run_one.py C2 1 > gpurun_out/k2_dram_C2_${TAG}_g$G.csv 2>&1
done
for G in 2 4 20 40; do
  BATMAP_K2_GROUP=$G timeout 600 ncu --metrics $M --clock-control none -k regex:k2_tiled -c 1 --csv python tools/run_one.py C4 1 > gpurun_out/k2_dram_C4_${TAG}_g$G.csv 2>&1
done
for f in gpurun_out/k2_dram_*_${TAG}_g*.csv; do echo $f; grep -E '"(dram__bytes_read.sum|gpu__time_duration.sum)"' $f | awk -F'","' '{print $(NF-2), $NF}'; done
