# ncu evidence for profiles/ (run under gpurun, one GPU):
#  1. launch list of the bench command (every launch, device time; cold-cache
#     and serialised, so compare shares, not absolutes)
#  2. --set full of the K2 scatter and K1 gather launches of the
#     device-resident loop (config 3 TP=1: 64 chunks x 80 layers, 5 GiB each)
#  3. --set full of the zero-copy/CE-path K2 (staging ring, one layer) and
#     K3 (one 32K-token chain)
set -x
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline \
  > gpurun_out/launches_bench.log 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:paged_copy -s 3 -c 2 \
  -o gpurun_out/prof_paged -f python bench.py --profile-kernels --steps 2 --warmup 1 \
  > gpurun_out/prof_paged.log 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:hash_chains -c 1 \
  -o gpurun_out/prof_hash -f python tools/bench_hash.py > gpurun_out/prof_hash.log 2>&1
# 4. --set full of the memo kernels on a warm 128K-token lookup (config 4)
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:"memo_|hash_chains" -s 12 -c 4 \
  -o gpurun_out/prof_memo -f python tools/bench_lookup.py > gpurun_out/prof_memo.log 2>&1
ls -la gpurun_out
