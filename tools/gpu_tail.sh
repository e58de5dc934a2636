mkdir -p gpurun_out
TAG=${TAG:-tail}
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.txt 2>&1; tail -2 gpurun_out/pytest_gpu_$TAG.txt
for v in 1 0 1; do BATMAP_K2_SPLIT=$v timeout 600 python bench.py --steps 10 --no-cpu-baseline --no-e2e > gpurun_out/bench_split${v}_$TAG.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/bench_split${v}_$TAG.json').read().strip().splitlines()[-1]); print('split=$v', round(d['ms_per_step'],3), round(d['phases_ms']['k2'],3), round(d['roofline']['frac'],4), d['gpu_launches'])"; done
timeout 1500 python tools/run_configs.py C1 C3 C5_p0.01 C4 > gpurun_out/configs_$TAG.jsonl 2>/dev/null
python -c "
import json
for l in open('gpurun_out/configs_$TAG.jsonl'):
    d=json.loads(l); print(d['config'], 'step', round(d['step_ms'],3), 'k2', round(d['k2_ms'],3), 'frac', round(d['k2_frac_R_int'] or 0,4), 'exact', d['exact'])"
