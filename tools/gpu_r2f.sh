# Build trace on C4; K2 tail via red.add: parity + timing + DRAM traffic; NEXT-4 bench.
mkdir -p gpurun_out
TAG=${TAG:-r2f}
BATMAP_TRACE=1 timeout 300 python tools/build_once.py C4 --n 3 > gpurun_out/trace_C4_$TAG.txt 2>&1; tail -24 gpurun_out/trace_C4_$TAG.txt
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c5_sweep.py -m gpu -q -x > gpurun_out/pytest_$TAG.txt 2>&1; tail -2 gpurun_out/pytest_$TAG.txt
timeout 900 python tools/run_configs.py C1 C2 C3 C5_p0.001 > gpurun_out/configs_$TAG.jsonl 2> gpurun_out/configs_$TAG.err; python -c "
import json
for l in open('gpurun_out/configs_$TAG.jsonl'):
    d=json.loads(l); print(d['config'], 'step %.3f k2 %.3f frac %.3f exact %s'%(d['step_ms'], d['k2_ms'], d['k2_frac_R_int'], d['exact']))
"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k2_tiled -s 2 -c 1 -o gpurun_out/k2_C2_$TAG python bench.py --config C2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-extra > gpurun_out/ncu_k2_C2_$TAG.log 2>&1; tail -1 gpurun_out/ncu_k2_C2_$TAG.log
timeout 900 python tools/triples_bench.py C3 C1 > gpurun_out/triples_bench_$TAG.jsonl 2> gpurun_out/triples_bench_$TAG.err; cat gpurun_out/triples_bench_$TAG.jsonl; tail -2 gpurun_out/triples_bench_$TAG.err
