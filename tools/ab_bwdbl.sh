for v in 0 1; do
  touch paper_2212_05159_b200/csrc/spgemm.cu
  CSRK_NVCC_EXTRA="-DCSRK_S_BWD_BL=$v" python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
  echo "BWD_BL=$v"; python tools/gemm_probe.py 2 | grep bwd; python tools/gemm_probe.py 3 | grep bwd
done
