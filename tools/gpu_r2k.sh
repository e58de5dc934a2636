# Round 2 (k): K2 time vs tile order (BATMAP_K2_GROUP=1 row-major vs the default bands), repeated.
mkdir -p gpurun_out
TAG=${TAG:-r2k}
for rep in 1 2; do
for cfg in C2 C5_p0.001 C5_p0.01 C4; do
  for G in 1 0 6 16; do
    BATMAP_K2_GROUP=$G timeout 300 python tools/run_one.py $cfg 3 >> gpurun_out/order_$TAG.txt 2>&1; echo "^ G=$G" >> gpurun_out/order_$TAG.txt
  done
done
done
cat gpurun_out/order_$TAG.txt
