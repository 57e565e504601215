# e2e variance across bench modes: 3 runs each, 5 timed steps.
mkdir -p gpurun_out
B="timeout 300 python bench.py --no-cpu-baseline --steps 5 --warmup 3"
for v in "" "--sequential"; do
  for r in 1 2 3; do
    $B $v > gpurun_out/m.json 2>>gpurun_out/m.err
    echo "[$v] run $r: $(python -c "import json; d=json.load(open('gpurun_out/m.json')); print(d['e2e']['value'], d['e2e']['ms_per_step'], d['links']['pcie']['bidir_gbps'])")"
  done
done
tail -2 gpurun_out/m.err
