# K1 tiers: build times per config (default tiers, and every r > 0 on the cluster kernel); then GPU tests
mkdir -p gpurun_out
TAG=${TAG:-k1}
timeout 600 python tools/build_bench.py C1 C2 C3 C4 C5_p0.01 C5_p0.05 C5_p0.1 > gpurun_out/build_$TAG.jsonl 2> gpurun_out/build_$TAG.err; tail -2 gpurun_out/build_$TAG.err
BATMAP_K1_SMALL=cluster timeout 600 python tools/build_bench.py C1 C2 > gpurun_out/build_allcluster_$TAG.jsonl 2>&1
BATMAP_K1_SMALL=legacy timeout 600 python tools/build_bench.py C1 C2 C3 C5_p0.01 > gpurun_out/build_legacy_$TAG.jsonl 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.txt 2>&1; tail -2 gpurun_out/pytest_gpu_$TAG.txt
