# Round 2 (ai): byte-tier tables staged item-major and transposed into the arena (BATMAP_K1_STAGE),
# A/B on the big-table classes, parity through the goldens / oracle, byte-tier GPU tests.
mkdir -p gpurun_out
TAG=${TAG:-r2ai}
timeout 900 python tools/build_bench.py --reps 7 --check --variants "byte=1;byte=1,stage=0" C5_p0.1 C5_p0.05 C4 C5_p0.01 > gpurun_out/build_$TAG.jsonl 2> gpurun_out/build_$TAG.err; python -c "
import json
for l in open('gpurun_out/build_$TAG.jsonl'):
    d=json.loads(l); print(d['config'], d['variant'], 'build %.2f k1 %.2f'%(d['build_ms'], d['k1_insert_ms']), 'exact', d.get('exact'))
"; tail -2 gpurun_out/build_$TAG.err
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c5_sweep.py -q -x > gpurun_out/pytest_$TAG.txt 2>&1; tail -2 gpurun_out/pytest_$TAG.txt
