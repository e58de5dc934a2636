# Round 2 (w): the triple kernel with batched loads -- parity, timing, ncu.
mkdir -p gpurun_out
TAG=${TAG:-r2w}
timeout 900 python -m pytest tests/test_gpu_triples.py -q -x > gpurun_out/pytest_triples_$TAG.txt 2>&1; tail -2 gpurun_out/pytest_triples_$TAG.txt
timeout 600 python tools/triples_bench.py --reps 5 C3 C1 > gpurun_out/triples_$TAG.jsonl 2> gpurun_out/triples_$TAG.err; cut -c1-700 gpurun_out/triples_$TAG.jsonl
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k3_triples -c 1 -o gpurun_out/k3t_C3_$TAG python tools/triples_bench.py --reps 1 --no-oracle C3 > gpurun_out/ncu_k3t_$TAG.log 2>&1; tail -1 gpurun_out/ncu_k3t_$TAG.log
# K2 tile width on C3 / C1 now that all-invalid blocks are skipped (the planner's choice uses whole tiles)
for tn in 64 128; do for cfg in C3 C1; do BATMAP_K2_TN=$tn timeout 120 python tools/run_one.py $cfg 7 >> gpurun_out/tn_$TAG.txt 2>&1; echo "tn=$tn" >> gpurun_out/tn_$TAG.txt; done; done; cat gpurun_out/tn_$TAG.txt
STRESS_SEED=77 timeout 500 python tools/stress.py 300 > gpurun_out/stress_$TAG.txt 2>&1; tail -1 gpurun_out/stress_$TAG.txt
