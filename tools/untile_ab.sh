#!/bin/bash
# A/B of the untile pass's frames per CTA (SRPGPU_UNTILE_FB) on cfg4 SSPI (gathered-window engine).
#   gpurun -- 'bash tools/untile_ab.sh'
mkdir -p gpurun_out
for fb in 1 4; do
  SRPGPU_UNTILE_FB=$fb timeout 600 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_scale.py -m gpu -k "tile" > gpurun_out/untile_tests_$fb.log 2>&1; echo "fb=$fb tests rc=$?"
done
for r in 1 2; do
  for fb in 1 2 4; do
    SRPGPU_UNTILE_FB=$fb timeout 600 python bench.py --workload cfg4 --no-variants --no-cpu-baseline --steps 3 --warmup 3 2>>gpurun_out/untile_ab.err \
      | sed "s/^/{\"fb\": $fb, \"r\": $r, \"line\": /; s/\$/}/" >> gpurun_out/untile_ab.jsonl
  done
done
