for cfg in "2 4" "3 5" "3 6" "2 6"; do
  set -- $cfg
  touch paper_2212_05159_b200/csrc/spmm.cu
  CSRK_NVCC_EXTRA="-DCSRK_WIDE_MINB_FWD=$1 -DCSRK_WIDE_MINB_DOT=$2" python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
  echo "FWD=$1 DOT=$2"; python tools/micro.py --ops spmm --reps 20 2>&1 | tail -1
done
