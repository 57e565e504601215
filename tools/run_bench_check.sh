mkdir -p gpurun_out
timeout 500 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --no-cpu-baseline --steps 1 --warmup 2 --trace > gpurun_out/trace.json 2>gpurun_out/trace.err
timeout 400 python bench.py > gpurun_out/bench.json 2>gpurun_out/bench.err; cat gpurun_out/bench.json; tail -2 gpurun_out/bench.err
