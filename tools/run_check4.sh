mkdir -p gpurun_out
timeout 500 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
timeout 400 python bench.py > gpurun_out/bench.json 2>gpurun_out/bench.err; cat gpurun_out/bench.json; tail -2 gpurun_out/bench.err
timeout 300 python bench.py --sequential --no-cpu-baseline > gpurun_out/bench_seq.json 2>>gpurun_out/bench.err; python -c "import json; d=json.load(open('gpurun_out/bench_seq.json')); print('sequential e2e', d['e2e'])"
timeout 900 python tools/bench_configs.py --only c4 2>&1 | tail -2
