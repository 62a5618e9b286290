# A/B of the 3xTF32 gathered-window kernel knobs (pair / one-CTA, fold chunk, unit group)
for P in 1 0; do for C in 2 4 8 64; do
  echo "pair=$P chunk=$C"; SRPGPU_GATHER_PAIR=$P SRPGPU_GATHER_CHUNK=$C timeout 300 python tools/bench_tile.py --fit fixed --engines tile 2>&1 | tail -1
done; done
