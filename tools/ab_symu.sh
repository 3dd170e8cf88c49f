#!/bin/bash
# A/B the lock-step width of the symmetric-pattern transpose (CSRK_SYM_U), config 2 + config 3 (3D).
cd "$(dirname "$0")/.."
for u in 1 2 4 8; do
  touch paper_2212_05159_b200/csrc/transpose.cu
  CSRK_NVCC_EXTRA="-DCSRK_SYM_U=$u" python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
  echo "U=$u $(python tools/micro.py --ops transpose --reps 20) $(python tools/micro.py --ops transpose --reps 20 --dim 3 --grid 160)"
done
touch paper_2212_05159_b200/csrc/transpose.cu
