for mb in 1 3 4; do
  touch paper_2212_05159_b200/csrc/sptrsv.cu paper_2212_05159_b200/csrc/radix.cu
  CSRK_NVCC_EXTRA="-DCSRK_LB_MINB=$mb -DCSRK_RS_MINB=$((mb+2))" python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
  echo "LB_MINB=$mb RS_MINB=$((mb+2))"
  python bench.py --workload trsv --steps 5 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print({k:v['ms'] for k,v in d['ops'].items()})"
  CSRK_TRANSPOSE_RADIX=1 python tools/micro.py --ops transpose --reps 10 2>&1 | tail -2
done
