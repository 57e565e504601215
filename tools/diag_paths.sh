# Host-tier path diagnosis: each direction alone and mixed, CE vs zero-copy store.
set -x
mkdir -p gpurun_out
timeout 400 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
B="timeout 300 python bench.py --no-cpu-baseline --steps 3 --warmup 2"
$B > gpurun_out/d_mixed_ce.json 2>gpurun_out/d.err
$B --store-zero-copy > gpurun_out/d_mixed_zc.json 2>>gpurun_out/d.err
$B --prefix 0 > gpurun_out/d_store_ce.json 2>>gpurun_out/d.err
$B --prefix 0 --store-zero-copy > gpurun_out/d_store_zc.json 2>>gpurun_out/d.err
$B --prefix 32768 > gpurun_out/d_load_ce.json 2>>gpurun_out/d.err
$B --prefix 32768 --load-zero-copy > gpurun_out/d_load_zc.json 2>>gpurun_out/d.err
for f in gpurun_out/d_*.json; do echo $f; python -c "import json,sys; d=json.load(open('$f')); print(d['e2e']['value'], d['e2e']['ms_per_step'], d['value'], d['roofline']['frac'])"; done
tail -5 gpurun_out/d.err
