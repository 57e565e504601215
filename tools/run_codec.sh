# q8 codec: GPU parity tests (both encode variants) and timing of each
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_codec.py -q -x -m gpu -p no:cacheprovider 2>&1 | tail -2
timeout 120 python tools/bench_codec.py 2>&1 | tail -1 | tee gpurun_out/codec.jsonl
TKV_Q8_ENCODE=twopass timeout 120 python tools/bench_codec.py 2>&1 | tail -1 | tee -a gpurun_out/codec.jsonl
