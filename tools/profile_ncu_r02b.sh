# ncu evidence for the late round-2 changes (run under gpurun, one GPU):
#  1. launch list of the bench command (after the affine K1/K2 form)
#  2. --set full of the unit kernel's affine one-layer launches (64 MiB / 8 MiB)
#  3. --set full of K3 after the a-chain rebuild (one 32K-token chain)
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --csv -c 3000 \
  --log-file gpurun_out/r02b_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-configs \
  > gpurun_out/r02b_launches_bench.log 2>&1
for b in 4096 512; do
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:paged_copy_units -s 200 -c 2 \
  -o gpurun_out/r02b_paged_affine_$b -f python tools/bench_k12_layers.py --bpt $b --reps 1 --affine \
  > gpurun_out/r02b_paged_affine_$b.log 2>&1
done
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:hash_chains_pair -c 1 \
  -o gpurun_out/r02b_k3 -f python tools/bench_hash.py > gpurun_out/r02b_k3.log 2>&1
for f in gpurun_out/r02b_paged_affine_4096 gpurun_out/r02b_paged_affine_512 gpurun_out/r02b_k3; do
  $NCU -i $f.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,launch__registers_per_thread 2>/dev/null | tail -n +2
done
