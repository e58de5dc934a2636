# Round 2 (s): full GPU suite + NEXT-4 timings + ncu of the grouped triple kernel.
mkdir -p gpurun_out
TAG=${TAG:-r2s}
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$TAG.txt 2>&1; tail -3 gpurun_out/pytest_gpu_$TAG.txt
timeout 600 python tools/triples_bench.py --reps 3 C3 C1 > gpurun_out/triples_$TAG.jsonl 2> gpurun_out/triples_$TAG.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k3_triples -c 1 -o gpurun_out/k3_triples_$TAG python tools/triples_bench.py --reps 1 C3 > gpurun_out/ncu_k3t_$TAG.log 2>&1
cut -c1-300 gpurun_out/triples_$TAG.jsonl
