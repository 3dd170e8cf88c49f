#!/bin/bash
# A/B the symbolic FILL copy kernel's CTA size / loads in flight (config 2 and 3 symbolic).
cd "$(dirname "$0")/.."
for f in ${FC:-"256 4" "256 6" "256 8" "512 8"}; do
  set -- $f
  touch paper_2212_05159_b200/csrc/spgemm.cu
  CSRK_NVCC_EXTRA="-DCSRK_FC_TPB=$1 -DCSRK_FC_BATCH=$2" python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
  echo "tpb=$1 batch=$2 $(python tools/micro.py --ops gemm --reps 20 | cut -c1-26) $(python tools/micro.py --ops gemm --reps 20 --dim 3 --grid 160 | cut -c1-26)"
done
touch paper_2212_05159_b200/csrc/spgemm.cu
