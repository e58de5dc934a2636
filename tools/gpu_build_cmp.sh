# K1 tiers: build times per config with the default tiers and with BATMAP_K1_SMALL=legacy|cluster; GPU tests
mkdir -p gpurun_out
TAG=${TAG:-k1}
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.txt 2>&1; tail -2 gpurun_out/pytest_gpu_$TAG.txt
timeout 600 python tools/build_bench.py C1 C2 C3 C4 C5_p0.01 C5_p0.05 C5_p0.1 > gpurun_out/build_$TAG.jsonl 2> gpurun_out/build_$TAG.err; tail -2 gpurun_out/build_$TAG.err
BATMAP_K1_SMALL=legacy timeout 600 python tools/build_bench.py C1 C2 C3 C5_p0.01 > gpurun_out/build_legacy_$TAG.jsonl 2>&1
BATMAP_K1_SMALL=cluster timeout 600 python tools/build_bench.py C1 C2 C3 C5_p0.01 > gpurun_out/build_cluster_$TAG.jsonl 2>&1
python - << 'PY'
import json, os
tag = os.environ.get("TAG", "k1")
for f in [f"gpurun_out/build_{tag}.jsonl", f"gpurun_out/build_legacy_{tag}.jsonl", f"gpurun_out/build_cluster_{tag}.jsonl"]:
    for l in open(f):
        try: d = json.loads(l)
        except Exception: continue
        print(f.split('/')[-1][:-6], d['config'], 'build', round(d['build_ms'], 3), 'ins', round(d['k1_insert_ms'], 3), 'fail', d['failures'])
PY
