# Round 2 (m): NEXT-4 launch list (where batmap3_build's time goes) on C3 and C1.
mkdir -p gpurun_out
TAG=${TAG:-r2m}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/triples_bench.py --reps 1 C3 > gpurun_out/launches_triples_C3_$TAG.csv 2>&1
timeout 600 python tools/triples_bench.py --reps 3 C3 C1 > gpurun_out/triples_$TAG.jsonl 2> gpurun_out/triples_$TAG.err
python tools/launch_summary.py gpurun_out/launches_triples_C3_$TAG.csv | head -30
cat gpurun_out/triples_$TAG.jsonl | cut -c1-400
