# Round 2 (ao): final re-measure after the staged pack in both K1 tiers -- every config, bench line (both arms),
# launch list, smoke.
mkdir -p gpurun_out
TAG=${TAG:-r2ao}
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.txt 2>&1; tail -1 gpurun_out/smoke_$TAG.txt
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -c 300 gpurun_out/bench_$TAG.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; tail -c 200 gpurun_out/bench_ref_$TAG.json
timeout 2400 python tools/run_configs.py > gpurun_out/configs_$TAG.jsonl 2> gpurun_out/configs_$TAG.err; tail -2 gpurun_out/configs_$TAG.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/launches_$TAG.log 2>&1; tail -c 200 gpurun_out/launches_$TAG.log
