#!/bin/bash
# compute-sanitizer over the kernels added / changed in round 2: the symmetric transpose (k_tr_sym)
# and the gated general path, the deterministic SpGEMM dB gather, k_rows with CTA-wide huge rows
# and the fused dot / accumulate modes (PCG), the GCN propagation / X^T dZ.  Caching allocator off.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
run() {  # tool, tag, pytest args...
  local tool=$1 tag=$2; shift 2
  PYTORCH_NO_CUDA_MEMORY_CACHING=1 timeout 1500 compute-sanitizer --tool $tool --print-limit 20 \
    python -m pytest "$@" -m gpu -x -q > gpurun_out/san_${tool}_$tag.log 2>&1
  echo "$tool $tag rc=$? | $(grep 'ERROR SUMMARY' gpurun_out/san_${tool}_$tag.log | tail -1) | $(grep -E 'passed|failed' gpurun_out/san_${tool}_$tag.log | tail -1)"
}
run memcheck parity tests/test_gpu_parity.py -k "transpose or spgemm or spmv"
run memcheck gcn tests/test_gpu_gcn.py
run memcheck pcg tests/test_pcg.py -k "not config5 and not slow and not fullsize and not full"
run racecheck parity tests/test_gpu_parity.py -k "symmetric or dB_plan or (spmv and (skew or powerlaw or poisson2d_70))"
run racecheck gcn tests/test_gpu_gcn.py -k "not bench"
run synccheck parity tests/test_gpu_parity.py -k "symmetric or dB_plan or (spmv and skew)"
