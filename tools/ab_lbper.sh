for per in 8 4 16; do
  touch paper_2212_05159_b200/csrc/sptrsv.cu
  CSRK_NVCC_EXTRA="-DCSRK_LB_PER=$per" python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
  echo "PER=$per"; python bench.py --workload trsv --steps 5 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print({k:v['ms'] for k,v in d['ops'].items() if 'chain' in k})"
done
