mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python tools/bench_configs.py --only c4 > gpurun_out/c4.jsonl 2>gpurun_out/c4.err; cat gpurun_out/c4.jsonl; tail -3 gpurun_out/c4.err
