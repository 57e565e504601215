# Validation: GPU tests, smoke, bench (default), reference arm, configs sweep (wall times recorded)
mkdir -p gpurun_out
t0=$(date +%s)
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
t1=$(date +%s); echo "pytest_gpu_s=$((t1-t0))"
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
t2=$(date +%s)
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2>gpurun_out/bench.err; cat gpurun_out/bench.json; tail -2 gpurun_out/bench.err
t3=$(date +%s); echo "bench_s=$((t3-t2))"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>gpurun_out/bench_ref.err; cat gpurun_out/bench_ref.json
t4=$(date +%s); echo "bench_ref_s(2+1 steps)=$((t4-t3))"
