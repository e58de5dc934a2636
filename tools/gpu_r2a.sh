# Round-2 first check: GPU tests (incl. the full C5 sweep), the default bench as the driver runs it, the reference arm.
mkdir -p gpurun_out
TAG=${TAG:-r2a}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi_$TAG.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.txt 2>&1; tail -1 gpurun_out/smoke_$TAG.txt
timeout 2400 python -m pytest tests -m gpu -q -x --durations=25 > gpurun_out/pytest_gpu_$TAG.txt 2>&1; tail -30 gpurun_out/pytest_gpu_$TAG.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -c 3000 gpurun_out/bench_$TAG.json; tail -3 gpurun_out/bench_$TAG.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; tail -c 600 gpurun_out/bench_ref_$TAG.json
