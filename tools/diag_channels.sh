mkdir -p gpurun_out
timeout 400 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
B="timeout 300 python bench.py --no-cpu-baseline --steps 3 --warmup 2"
for c in 8 32; do
  CUDA_DEVICE_MAX_CONNECTIONS=$c $B > gpurun_out/c_mixed_$c.json 2>>gpurun_out/c.err
  echo "conn=$c mixed: $(python -c "import json; d=json.load(open('gpurun_out/c_mixed_$c.json')); print(d['e2e']['value'], d['e2e']['ms_per_step'])")"
done
CUDA_DEVICE_MAX_CONNECTIONS=32 $B --store-zero-copy > gpurun_out/c_mixed_zc32.json 2>>gpurun_out/c.err
echo "conn=32 mixed zc: $(python -c "import json; d=json.load(open('gpurun_out/c_mixed_zc32.json')); print(d['e2e']['value'], d['e2e']['ms_per_step'])")"
tail -3 gpurun_out/c.err
