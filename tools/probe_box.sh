set -x
nvidia-smi; nvidia-smi topo -m; free -g; nproc; lscpu | head -30; numactl -H 2>/dev/null | head; cat /proc/meminfo | head -5; ulimit -a
mkdir -p gpurun_out
./build/microbench 2>&1 | tee gpurun_out/microbench.txt
