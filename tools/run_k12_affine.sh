# K1/K2 one-layer launches: descriptor-list unit kernel vs the affine form; GPU parity of the paths
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_connector.py tests/test_gpu_pipeline.py -q -x -m gpu -p no:cacheprovider 2>&1 | tail -2
timeout 300 python tools/bench_k12_layers.py --bpt 4096 1024 512 2>&1 | grep -E '"K1 gather"|"K2 scatter"' | tee gpurun_out/k12_layers.jsonl
timeout 300 python tools/bench_k12_layers.py --bpt 4096 1024 512 --affine 2>&1 | grep -E '"K1 gather"|"K2 scatter"' | tee -a gpurun_out/k12_layers.jsonl
