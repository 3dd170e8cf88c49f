#!/bin/bash
# compute-sanitizer memcheck over the small GPU parity cases (one process per test file); torch's
# caching allocator is off so that every tensor is its own allocation (memcheck sees overruns).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for f in tests/test_gpu_parity.py tests/test_gpu_spadd.py tests/test_gpu_sptrsv.py tests/test_gpu_gcn.py tests/test_gpu_radix.py; do
  b=$(basename $f .py)
  PYTORCH_NO_CUDA_MEMORY_CACHING=1 timeout 1500 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 --print-limit 20 \
    python -m pytest $f -m gpu -x -q -k "not big and not fullsize and not bench and not huge" > gpurun_out/memcheck_$b.log 2>&1
  echo "$b rc=$? $(grep -c 'Invalid\|ERROR SUMMARY: [1-9]' gpurun_out/memcheck_$b.log) $(grep 'ERROR SUMMARY' gpurun_out/memcheck_$b.log | tail -1) $(tail -1 gpurun_out/memcheck_$b.log)"
done
for f in tests/test_pcg.py tests/test_spai.py tests/test_gpu_validate.py; do
  b=$(basename $f .py)
  PYTORCH_NO_CUDA_MEMORY_CACHING=1 timeout 1500 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 --print-limit 20 \
    python -m pytest $f -m gpu -x -q -k "not config5 and not slow and not fullsize" > gpurun_out/memcheck_$b.log 2>&1
  echo "$b rc=$? $(grep 'ERROR SUMMARY' gpurun_out/memcheck_$b.log | tail -1) $(grep -E 'passed|failed' gpurun_out/memcheck_$b.log | tail -1)"
done
PYTORCH_NO_CUDA_MEMORY_CACHING=1 compute-sanitizer --tool memcheck --print-limit 1 python tools/sanitizer_selftest.py > gpurun_out/memcheck_selftest.log 2>&1
echo "selftest (must report errors): $(grep 'ERROR SUMMARY' gpurun_out/memcheck_selftest.log | tail -1)"
