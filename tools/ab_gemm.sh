bash tools/gpu_check.sh "sptrsv or spmv or transpose or config4 or gcn" "trsv cfg4 cfg2"
grep -E "Error|Mismatch|FAILED" gpurun_out/gputests.log | head -10
for mb in 1 4 6; do
  touch paper_2212_05159_b200/csrc/spgemm.cu
  CSRK_NVCC_EXTRA="-DCSRK_S_MINB=$mb" python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
  echo "MINB=$mb"; python tools/gemm_probe.py 2
done
