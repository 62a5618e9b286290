# tile-chunk unit order: DRAM bytes / time of the fp16x3 pair kernel (cfg4, fixed fit, 10^4 frames)
run() { env "$@" timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k "regex:gather_pair" -s 1 -c 1 --csv python tools/prof_chain.py --workload cfg4 --variant sspi --frames 10000 --reps 2 --engine tile_f16 2>/dev/null | grep gather_pair | rev | cut -d, -f1-3 | rev | tr '\n' ' '; echo " <- $*"; }
run SRPGPU_GATHER_TCHUNK=18 SRPGPU_GATHER_GROUP=1024 SRPGPU_GATHER_L2=2
run SRPGPU_GATHER_TCHUNK=37 SRPGPU_GATHER_GROUP=512 SRPGPU_GATHER_L2=2
run SRPGPU_GATHER_TCHUNK=18 SRPGPU_GATHER_GROUP=1024 SRPGPU_GATHER_L2=0
run SRPGPU_GATHER_TCHUNK=18 SRPGPU_GATHER_GROUP=1024 SRPGPU_GATHER_L2=1
run SRPGPU_GATHER_TCHUNK=9 SRPGPU_GATHER_GROUP=2048 SRPGPU_GATHER_L2=2
run SRPGPU_GATHER_TCHUNK=36 SRPGPU_GATHER_GROUP=1024 SRPGPU_GATHER_L2=2
