# Round 2 (an): staged pack for the uint32 CTA tier too -- A/B with parity, GPU suite.
mkdir -p gpurun_out
TAG=${TAG:-r2an}
timeout 1200 python tools/build_bench.py --reps 7 --check --variants "byte=1;byte=1,stage=0" C5_p0.02 C5_p0.01 C5_p0.005 C5_p0.1 C4 C3 C2 > gpurun_out/build_$TAG.jsonl 2> gpurun_out/build_$TAG.err; python -c "
import json
for l in open('gpurun_out/build_$TAG.jsonl'):
    d=json.loads(l); print(d['config'], d['variant'], 'build %.2f k1 %.2f'%(d['build_ms'], d['k1_insert_ms']), 'exact', d.get('exact'))
"; tail -2 gpurun_out/build_$TAG.err
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$TAG.txt 2>&1; tail -2 gpurun_out/pytest_gpu_$TAG.txt
STRESS_SEED=555 timeout 400 python tools/stress.py 240 > gpurun_out/stress_$TAG.txt 2>&1; tail -1 gpurun_out/stress_$TAG.txt
