#!/bin/bash
# memcheck over the bench-size parity tests (config 2 / 3 / 4 at full size), caching allocator off.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for k in config2 config3 config4; do
  PYTORCH_NO_CUDA_MEMORY_CACHING=1 timeout 1500 compute-sanitizer --tool memcheck --leak-check no --print-limit 20 \
    python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -k $k > gpurun_out/memcheck_full_$k.log 2>&1
  echo "memcheck_full_$k rc=$? $(grep -E 'passed|failed' gpurun_out/memcheck_full_$k.log | tail -1) | $(grep 'ERROR SUMMARY' gpurun_out/memcheck_full_$k.log | tail -1)"
done
