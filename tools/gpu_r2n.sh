# Round 2 (n): NEXT-4 build (chunked encode, pooled buffers), warp-per-candidate corrections, pair-grouped triple kernel.
mkdir -p gpurun_out
TAG=${TAG:-r2n}
timeout 900 python -m pytest tests/test_gpu_triples.py -q -x > gpurun_out/pytest_triples_$TAG.txt 2>&1; tail -3 gpurun_out/pytest_triples_$TAG.txt
timeout 600 python tools/triples_bench.py --reps 3 C3 C1 > gpurun_out/triples_$TAG.jsonl 2> gpurun_out/triples_$TAG.err
BATMAP_K3_GROUPED=0 timeout 600 python tools/triples_bench.py --reps 3 C3 > gpurun_out/triples_${TAG}_ungrouped.jsonl 2>> gpurun_out/triples_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/triples_bench.py --reps 1 C3 > gpurun_out/launches_triples_C3_$TAG.csv 2>&1
grep -v "^==\|^{" gpurun_out/launches_triples_C3_$TAG.csv > gpurun_out/launches_triples_C3_$TAG.clean.csv
python tools/launch_summary.py gpurun_out/launches_triples_C3_$TAG.clean.csv > gpurun_out/launches_triples_C3_$TAG.txt; head -16 gpurun_out/launches_triples_C3_$TAG.txt
cut -c1-420 gpurun_out/triples_$TAG.jsonl gpurun_out/triples_${TAG}_ungrouped.jsonl; tail -3 gpurun_out/triples_$TAG.err
