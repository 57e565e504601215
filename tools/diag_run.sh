mkdir -p gpurun_out
timeout 500 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --no-cpu-baseline --steps 1 --warmup 2 --trace > gpurun_out/trace.json 2>gpurun_out/trace.err
B="timeout 300 python bench.py --no-cpu-baseline --steps 3 --warmup 2"
for v in "" "--store-zero-copy"; do
  $B $v > gpurun_out/m.json 2>>gpurun_out/m.err
  echo "mixed [$v]: $(python -c "import json; d=json.load(open('gpurun_out/m.json')); print(d['e2e']['value'], d['e2e']['ms_per_step'], d['value'])")"
done
tail -3 gpurun_out/m.err
