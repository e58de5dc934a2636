# Round 2 (ac): final verification at HEAD -- GPU suite, stress (balanced mode randomised), part
# balance of the final planner, bench line.
mkdir -p gpurun_out
TAG=${TAG:-r2ac}
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$TAG.txt 2>&1; tail -2 gpurun_out/pytest_gpu_$TAG.txt
STRESS_SEED=4242 timeout 900 python tools/stress.py 720 > gpurun_out/stress_$TAG.txt 2>&1; tail -1 gpurun_out/stress_$TAG.txt
timeout 1500 python tools/part_balance.py C4 C5_p0.1 C5_p0.01 C2 > gpurun_out/part_balance_$TAG.jsonl 2> gpurun_out/part_balance_$TAG.err; cut -c1-200 gpurun_out/part_balance_$TAG.jsonl
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -c 300 gpurun_out/bench_$TAG.json
