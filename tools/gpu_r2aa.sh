# Round 2 (aa): split-K granularity and the finer cut of accumulated tail pieces, re-measured with
# K2's balanced mode on (C3, C1 are all split-K / accumulated).
mkdir -p gpurun_out
TAG=${TAG:-r2aa}
for rep in 1 2; do for f in 2 3 4 6 8; do for at in 1 0; do for cfg in C3 C1; do
  echo -n "f=$f acctail=$at " >> gpurun_out/split_$TAG.txt
  BATMAP_K2_SPLITF=$f BATMAP_K2_ACCTAIL=$at timeout 120 python tools/run_one.py $cfg 9 >> gpurun_out/split_$TAG.txt 2>&1
done; done; done; done
cat gpurun_out/split_$TAG.txt
