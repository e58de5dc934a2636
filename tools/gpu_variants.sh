mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "c1 or mixed or c2_full or items" > gpurun_out/pytest_var.txt 2>&1; tail -2 gpurun_out/pytest_var.txt
for v in ${VARIANTS:-0 1}; do
  BATMAP_K2_VARIANT=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_v$v.json 2>gpurun_out/bench_v$v.err
  python -c "import json;d=json.load(open('gpurun_out/bench_v$v.json'));r=d['roofline'];print('variant $v', round(d['value']/1e9,3),'Gpairs/s', 'k2_ms',round(r['k2_ms'],3),'frac',round(r['frac'],4), 'build', round(d['phases_ms']['build'],3))" || tail -5 gpurun_out/bench_v$v.err
done
