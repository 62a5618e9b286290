timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "sspi_and_si or engines_agree" 2>&1 | tail -2
for G in 512 1024 2048; do
  echo "group=$G"; SRPGPU_GATHER_GROUP=$G timeout 300 python tools/bench_tile.py --fit fixed --engines tile 2>&1 | tail -1
done
