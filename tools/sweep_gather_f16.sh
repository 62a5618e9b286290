# A/B of the pair kernel's map store paths and chunk sizes (fixed fit, cfg4, fp16x3)
run() { env "$@" timeout 900 python tools/bench_tile.py --fit fixed --engines tile_f16 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$*', d['map_ms'], d['map_argmax_only_ms'], d['err'], d['argmax_agree'])"; }
run A=0
run SRPGPU_GATHER_ZSTG=1
run SRPGPU_GATHER_CHUNK=16
run SRPGPU_UNTILE_FB=2
