#!/bin/bash
# A/B the SpMM pipelined path's L2 prefetch distance (CSRK_SPMM_PF_FWD / _DOT) on config 2.
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
for pf in 0 1 2 3 4 6; do
  echo "pf=$pf $(CSRK_SPMM_PF_FWD=$pf CSRK_SPMM_PF_DOT=$pf python tools/micro.py --ops spmm --reps 20)"
done
