# Round 2 (ad): hoisted-parameter triple kernel (4 or 8 candidates per CTA) vs the grouped kernel.
mkdir -p gpurun_out
TAG=${TAG:-r2ad}
for h in 4 8; do BATMAP_K3_HOIST=$h timeout 900 python -m pytest tests/test_gpu_triples.py -q -x > gpurun_out/pytest_triples_h${h}_$TAG.txt 2>&1; echo "hoist=$h $(tail -1 gpurun_out/pytest_triples_h${h}_$TAG.txt)"; done
for rep in 1 2; do for h in 0 4 8; do
  BATMAP_K3_HOIST=$h timeout 600 python tools/triples_bench.py --reps 5 --no-oracle C3 C1 > gpurun_out/tri_h${h}_${rep}_$TAG.jsonl 2>/dev/null
  python -c "
import json,sys
for l in open('gpurun_out/tri_h${h}_${rep}_$TAG.jsonl'):
    d=json.loads(l); print('hoist=$h', d['config'], 'kernel %.3f ms'%d['triples_kernel_ms'], 'K3', d['frequent_triples'])
" >> gpurun_out/tri_ab_$TAG.txt
done; done
cat gpurun_out/tri_ab_$TAG.txt
