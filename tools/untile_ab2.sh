# untile pass A/B on the blocked scratch (cfg4, fixed fit): frames per CTA
run() { env "$@" timeout 900 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k "regex:untile" -s 1 -c 1 --csv python tools/prof_chain.py --workload cfg4 --variant sspi --frames 10000 --reps 2 --engine tile_f16 2>/dev/null | grep untile | rev | cut -d, -f1-3 | rev | tr '\n' ' '; echo " <- $*"; }
run SRPGPU_UNTILE_FB=4
run SRPGPU_UNTILE_FB=8
run SRPGPU_UNTILE_FB=2
