# Round 2 (ae): hoisted triple kernel, candidates per CTA 2 / 4 / 6 (default 4), and on C1's narrow
# BatMaps (BATMAP_K3_GROUPED=1); triples parity with the default.
mkdir -p gpurun_out
TAG=${TAG:-r2ae}
timeout 900 python -m pytest tests/test_gpu_triples.py -q -x > gpurun_out/pytest_triples_$TAG.txt 2>&1; tail -1 gpurun_out/pytest_triples_$TAG.txt
BATMAP_K3_GROUPED=1 timeout 900 python -m pytest tests/test_gpu_triples.py -q -x > gpurun_out/pytest_triples_g1_$TAG.txt 2>&1; tail -1 gpurun_out/pytest_triples_g1_$TAG.txt
for rep in 1 2; do for h in 2 4 6; do for g in "" 1; do
  BATMAP_K3_HOIST=$h BATMAP_K3_GROUPED=$g timeout 600 python tools/triples_bench.py --reps 5 --no-oracle C3 C1 > gpurun_out/tri_${h}_${g}_${rep}_$TAG.jsonl 2>/dev/null
  python -c "
import json
for l in open('gpurun_out/tri_${h}_${g}_${rep}_$TAG.jsonl'):
    d=json.loads(l); print('hoist=$h grouped=${g:-default}', d['config'], 'kernel %.3f ms'%d['triples_kernel_ms'], 'K3', d['frequent_triples'])
" >> gpurun_out/tri_ab_$TAG.txt
done; done; done
cat gpurun_out/tri_ab_$TAG.txt
timeout 600 python tools/triples_bench.py --reps 5 C3 C1 > gpurun_out/triples_$TAG.jsonl 2> gpurun_out/triples_$TAG.err; cut -c1-400 gpurun_out/triples_$TAG.jsonl
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k3_triples -c 1 -o gpurun_out/k3t_C3_$TAG python tools/triples_bench.py --reps 1 --no-oracle C3 > gpurun_out/ncu_k3t_$TAG.log 2>&1; tail -1 gpurun_out/ncu_k3t_$TAG.log
