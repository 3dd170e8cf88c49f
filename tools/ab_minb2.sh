for mb in 6 8 10; do
  touch paper_2212_05159_b200/csrc/spgemm.cu
  CSRK_NVCC_EXTRA="-DCSRK_S_MINB=$mb" python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
  echo "MINB=$mb"; python tools/gemm_probe.py 2; python tools/gemm_probe.py 3
done
