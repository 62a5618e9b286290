#!/bin/bash
# Round-end check on one B200: GPU tests, smoke(), the default bench line.
#   gpurun -- 'bash tools/final_check.sh'
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/final_gpu_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/final_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/final_bench.jsonl 2> gpurun_out/final_bench.err; echo "bench rc=$?"
