# Round 2 (t): re-measure at HEAD after the container restore: GPU suite, bench (both arms),
# every config incl. all 7 C5 points vs the full-size goldens, launch list, ncu of K2 / K1.
mkdir -p gpurun_out
TAG=${TAG:-r2t}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi_$TAG.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.txt 2>&1; tail -1 gpurun_out/smoke_$TAG.txt
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/pytest_gpu_$TAG.txt 2>&1; tail -2 gpurun_out/pytest_gpu_$TAG.txt
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -c 400 gpurun_out/bench_$TAG.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; tail -c 300 gpurun_out/bench_ref_$TAG.json
timeout 2400 python tools/run_configs.py ${CONFIGS:-C1 C2 C3 C4 C5_p0.001 C5_p0.002 C5_p0.005 C5_p0.01 C5_p0.02 C5_p0.05 C5_p0.1} > gpurun_out/configs_$TAG.jsonl 2> gpurun_out/configs_$TAG.err; tail -3 gpurun_out/configs_$TAG.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/launches_$TAG.log 2>&1; tail -2 gpurun_out/launches_$TAG.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k2_tiled -s 3 -c 1 -o gpurun_out/k2_full_$TAG python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-extra > gpurun_out/ncu_$TAG.log 2>&1; tail -2 gpurun_out/ncu_$TAG.log
timeout 900 ncu --set full --clock-control none -k regex:k1_ -c 6 -o gpurun_out/k1_full_$TAG python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-extra > gpurun_out/ncu_k1_$TAG.log 2>&1; tail -2 gpurun_out/ncu_k1_$TAG.log
