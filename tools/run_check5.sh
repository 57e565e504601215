mkdir -p gpurun_out
B="timeout 300 python bench.py --no-cpu-baseline --steps 3 --warmup 2"
for v in "" "--memo-entries 0" "--sequential --memo-entries 0"; do
  $B $v > gpurun_out/m.json 2>>gpurun_out/m.err
  echo "[$v]: $(python -c "import json; d=json.load(open('gpurun_out/m.json')); print(d['e2e']['value'], d['e2e']['ms_per_step'])")"
done
timeout 300 python bench.py --no-cpu-baseline --steps 1 --warmup 2 --trace --memo-entries 0 > gpurun_out/trace.json 2>>gpurun_out/m.err; cat gpurun_out/trace.json
tail -3 gpurun_out/m.err
timeout 300 python tools/bench_hash.py 2>&1 | head -3
