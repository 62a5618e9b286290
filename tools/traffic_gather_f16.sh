# DRAM bytes of the fp16x3 pair kernel (cfg4, fixed fit, 10^4 frames) under L2 policy / frame-group settings
# SRPGPU_GATHER_L2: bits 0-1 samples, 2-3 slabs, 4-5 map stores (0 evict_last|first(stores), 1 evict_first|normal(stores), 2 evict_normal|last(stores))
run() { env "$@" timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k "regex:gather_pair" -s 1 -c 1 --csv python tools/prof_chain.py --workload cfg4 --variant sspi --frames 10000 --reps 2 --engine tile_f16 2>/dev/null | grep gather_pair | rev | cut -d, -f1-3 | rev | tr '\n' ' '; echo " <- $*"; }
run A=0
run SRPGPU_GATHER_L2=24
run SRPGPU_GATHER_GROUP=2048
run SRPGPU_GATHER_GROUP=2048 SRPGPU_GATHER_L2=0
run SRPGPU_GATHER_GROUP=512
run SRPGPU_GATHER_L2=4
