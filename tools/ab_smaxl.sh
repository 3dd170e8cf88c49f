for ml in 8 6 4; do
  touch paper_2212_05159_b200/csrc/spgemm.cu
  CSRK_NVCC_EXTRA="-DCSRK_S_MAXL=$ml" python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
  echo "S_MAXL=$ml"; python tools/gemm_probe.py 3; python tools/gemm_probe.py 2
done
