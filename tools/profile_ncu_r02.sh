# ncu evidence for round 2 (run under gpurun, one GPU; outputs in gpurun_out/):
#  1. launch list of the bench command (device time of every launch; cold-cache
#     and serialised under ncu, so compare shares, not absolutes)
#  2. --set full of the tile kernel's all-layer K2 / K1 (the roofline kernel of
#     bench.py's value loop: config 3 TP=1, 5 GiB per launch)
#  3. --set full of the unit kernel on one-layer launches (the layerwise
#     connector's K2 / K1: 64 MiB at bpt 4096, 8 MiB at bpt 512)
#  4. --set full of K3 (one 32K-token chain: hash_chains_pair_kernel)
#  5. --set full of the lookup kernels: first_row_kernel (cold document) and
#     the memo probe / fingerprint / verify kernels (stored document)
set -x
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --csv -c 3000 \
  --log-file gpurun_out/r02_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-configs \
  > gpurun_out/r02_launches_bench.log 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:paged_copy_kernel -s 3 -c 2 \
  -o gpurun_out/r02_paged_tile -f python bench.py --profile-kernels --steps 2 --warmup 1 \
  > gpurun_out/r02_paged_tile.log 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:paged_copy_units -s 200 -c 2 \
  -o gpurun_out/r02_paged_units_4096 -f python tools/bench_k12_layers.py --bpt 4096 --reps 1 \
  > gpurun_out/r02_paged_units_4096.log 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:paged_copy_units -s 200 -c 2 \
  -o gpurun_out/r02_paged_units_512 -f python tools/bench_k12_layers.py --bpt 512 --reps 1 \
  > gpurun_out/r02_paged_units_512.log 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:hash_chains_pair -c 1 \
  -o gpurun_out/r02_k3 -f python tools/bench_hash.py > gpurun_out/r02_k3.log 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:"first_row|memo_|presence" -s 20 -c 8 \
  -o gpurun_out/r02_lookup -f python tools/bench_lookup.py > gpurun_out/r02_lookup.log 2>&1
ls -la gpurun_out
