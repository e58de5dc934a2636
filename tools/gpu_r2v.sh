# Round 2 (v): randomized exactness stress on the round-2 code (byte-table K1 tier randomised, NEXT-4
# triples path vs horizontal triple counting), ncu source capture of C2's K2.
mkdir -p gpurun_out
TAG=${TAG:-r2v}
STRESS_SEED=2026 timeout 1300 python tools/stress.py ${STRESS_S:-1100} > gpurun_out/stress_$TAG.txt 2>&1; tail -2 gpurun_out/stress_$TAG.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k2_tiled -s 2 -c 1 -o gpurun_out/k2_C2_$TAG python tools/run_one.py C2 3 > gpurun_out/ncu_k2c2_$TAG.log 2>&1; tail -1 gpurun_out/ncu_k2c2_$TAG.log
