# Round 2 (l): tail cut of accumulated k-pieces + row-major for L2-sized rectangles: GPU tests,
# configs, K2 DRAM traffic on C2 / C3, C3 launch list.
mkdir -p gpurun_out
TAG=${TAG:-r2l}
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$TAG.txt 2>&1; tail -3 gpurun_out/pytest_gpu_$TAG.txt
timeout 2000 python tools/run_configs.py C1 C2 C3 C4 C5_p0.001 C5_p0.1 > gpurun_out/configs_$TAG.jsonl 2> gpurun_out/configs_$TAG.err; tail -2 gpurun_out/configs_$TAG.err
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct
for cfg in C2 C3; do
  timeout 300 ncu --metrics $M --clock-control none -k regex:k2_tiled -c 1 --csv python tools/run_one.py $cfg 1 > gpurun_out/k2_dram_${cfg}_$TAG.csv 2>&1
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/run_one.py C3 2 > gpurun_out/launches_C3_$TAG.csv 2>&1
grep -h '"dram__bytes_read.sum"\|"gpu__time_duration.sum"' gpurun_out/k2_dram_*_$TAG.csv | awk -F'","' '{print $(NF-2), $NF}'
