# Round 2 (aj): staged byte-tier pack for IPC <= 2 (default) / <= 4 / off, A/B with parity checks.
mkdir -p gpurun_out
TAG=${TAG:-r2aj}
timeout 1200 python tools/build_bench.py --reps 7 --check --variants "byte=1;byte=1,stage=4;byte=1,stage=0" C5_p0.1 C5_p0.05 C5_p0.02 C5_p0.01 C4 C2 C3 > gpurun_out/build_$TAG.jsonl 2> gpurun_out/build_$TAG.err; python -c "
import json
for l in open('gpurun_out/build_$TAG.jsonl'):
    d=json.loads(l); print(d['config'], d['variant'], 'build %.2f k1 %.2f'%(d['build_ms'], d['k1_insert_ms']), 'exact', d.get('exact'))
"; tail -2 gpurun_out/build_$TAG.err
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$TAG.txt 2>&1; tail -2 gpurun_out/pytest_gpu_$TAG.txt
