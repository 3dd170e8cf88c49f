for u in 4 8 2; do
  touch paper_2212_05159_b200/csrc/spmv.cu paper_2212_05159_b200/csrc/transpose.cu
  CSRK_NVCC_EXTRA="-DCSRK_STREAM_UNROLL=$u" python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
  echo "UNROLL=$u"; python bench.py --steps 5 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print({k:v['ms'] for k,v in d['ops'].items() if k in ('csr_transpose','spmv_fwd','spmv_bwd')})"
done
