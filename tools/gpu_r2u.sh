# Round 2 (u): after the planner change -- GPU suite, build timings, part balance at N = 2/4/8,
# ncu of C3's K2 and of the triple kernel, the four sanitizers on the extended case (byte-table K1, NEXT-4).
mkdir -p gpurun_out
TAG=${TAG:-r2u}
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$TAG.txt 2>&1; tail -2 gpurun_out/pytest_gpu_$TAG.txt
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -c 300 gpurun_out/bench_$TAG.json
timeout 600 python tools/build_bench.py --reps 7 C2 C3 C4 C5_p0.01 C5_p0.1 > gpurun_out/build_$TAG.jsonl 2> gpurun_out/build_$TAG.err; cut -c1-200 gpurun_out/build_$TAG.jsonl
BATMAP_TRACE=1 timeout 300 python tools/run_one.py C4 3 > gpurun_out/trace_c4_$TAG.txt 2>&1; tail -9 gpurun_out/trace_c4_$TAG.txt
timeout 1200 python tools/part_balance.py C4 C5_p0.1 C2 > gpurun_out/part_balance_$TAG.jsonl 2> gpurun_out/part_balance_$TAG.err; cut -c1-300 gpurun_out/part_balance_$TAG.jsonl
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k2_tiled -s 2 -c 1 -o gpurun_out/k2_C3_$TAG python tools/run_one.py C3 3 > gpurun_out/ncu_k2c3_$TAG.log 2>&1; tail -1 gpurun_out/ncu_k2c3_$TAG.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k3_triples -c 1 -o gpurun_out/k3t_C3_$TAG python tools/triples_bench.py --reps 1 --no-oracle C3 > gpurun_out/ncu_k3t_$TAG.log 2>&1; tail -1 gpurun_out/ncu_k3t_$TAG.log
for tool in memcheck racecheck synccheck initcheck; do
  SANITIZE_TOOL=$tool timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_case.py > gpurun_out/sanitize_${tool}_$TAG.txt 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|sanitize case" gpurun_out/sanitize_${tool}_$TAG.txt | head -3
done
