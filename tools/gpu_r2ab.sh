# Round 2 (ab): K2 inner chunk loop unrolled by 2 for 128-wide tiles -- A/B against the previous
# library (tmp_ab/libbatmap_old.so), then the GPU suite on the new one.
mkdir -p gpurun_out
TAG=${TAG:-r2ab}
cp paper_1102_1003_b200/libbatmap.so tmp_ab/libbatmap_new.so
for rep in 1 2 3; do for v in new old; do
  cp tmp_ab/libbatmap_$v.so paper_1102_1003_b200/libbatmap.so
  for cfg in C2 C5_p0.001; do echo -n "$v " >> gpurun_out/unroll_$TAG.txt; timeout 300 python tools/run_one.py $cfg 9 >> gpurun_out/unroll_$TAG.txt 2>&1; done
done; done
cp tmp_ab/libbatmap_new.so paper_1102_1003_b200/libbatmap.so
cat gpurun_out/unroll_$TAG.txt
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$TAG.txt 2>&1; tail -2 gpurun_out/pytest_gpu_$TAG.txt
