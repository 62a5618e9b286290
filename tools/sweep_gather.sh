# DRAM traffic of the 3xTF32 pair kernel by unit group and L2 policies (samples | slabs << 2;
# 0 evict_last, 1 evict_first, 2 evict_normal)
run() { echo "group=$1 l2=$2"; SRPGPU_GATHER_GROUP=$1 SRPGPU_GATHER_L2=$2 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"gather" -c 1 python tools/bench_tile.py --fit fixed --engines tile --frames 4096 2>&1 | grep -E "duration|dram" | awk '{print $1, $3}' | paste - -; }
run 1024 4; run 512 4; run 2048 4; run 1024 8; run 1024 0; run 1024 10; run 1024 5
