#!/bin/bash
# A/B the occupancy hint of the pipelined SpMM kernel (CTAs of 128 threads per SM), config 2.
cd "$(dirname "$0")/.."
for f in ${PAIRS:-"4 3" "4 4"}; do
  set -- $f
  touch paper_2212_05159_b200/csrc/spmm.cu
  CSRK_NVCC_EXTRA="-DCSRK_PIPE_MINB_FWD=$1 -DCSRK_PIPE_MINB_DOT=$2" python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
  echo "fwd=$1 dot=$2 $(python tools/micro.py --ops spmm --reps 20)"
done
touch paper_2212_05159_b200/csrc/spmm.cu
