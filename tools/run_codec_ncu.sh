mkdir -p gpurun_out
TKV_Q8_CFG=${CFG:-4} timeout 300 ncu --set full --import-source on --clock-control none -k regex:q8_encode_fused -c 1 -o gpurun_out/q8_fused -f python tools/bench_codec.py > /dev/null 2>&1
ncu -i gpurun_out/q8_fused.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct 2>&1 | tail -1
