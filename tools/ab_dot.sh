#!/bin/bash
# A/B of the fused SpMM backward variants on config 2 (runtime knobs).
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
for v in "X=0" "CSRK_SPMM_G8_DOT=1" "CSRK_SPMM_PIPE_W=1" "CSRK_SPMM_L1_DOT=1" "CSRK_SPMM_G8_FWD=1" "CSRK_SPMM_L1_FWD=1" "CSRK_SPMM_PIPE=0"; do
  echo "$v $(env $v python tools/micro.py --ops spmm --reps 20)"
done
