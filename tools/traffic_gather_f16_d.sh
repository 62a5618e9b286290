run() { env "$@" timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k "regex:gather_pair" -s 1 -c 1 --csv python tools/prof_chain.py --workload cfg4 --variant sspi --frames 10000 --reps 2 --engine tile_f16 2>/dev/null | grep gather_pair | rev | cut -d, -f1-3 | rev | tr '\n' ' '; echo " <- $*"; }
run A=0
run SRPGPU_GATHER_L2=8 SRPGPU_GATHER_GROUP=512
run SRPGPU_GATHER_L2=6 SRPGPU_GATHER_GROUP=512
run SRPGPU_GATHER_L2=5 SRPGPU_GATHER_GROUP=512
