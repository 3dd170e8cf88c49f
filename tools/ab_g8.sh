#!/bin/bash
# A/B the 8-lanes-per-row pipelined SpMM (CSRK_SPMM_G8_DOT / _FWD) at several occupancy hints.
cd "$(dirname "$0")/.."
for mb in 3 4; do
  touch paper_2212_05159_b200/csrc/spmm.cu
  CSRK_NVCC_EXTRA="-DCSRK_PIPE_MINB_G8=$mb" python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
  echo "G8 minb=$mb $(CSRK_SPMM_G8_DOT=1 CSRK_SPMM_G8_FWD=1 python tools/micro.py --ops spmm --reps 20)"
done
touch paper_2212_05159_b200/csrc/spmm.cu
