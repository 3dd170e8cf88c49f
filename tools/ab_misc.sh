for cfg in "1 1" "8 8" "6 12"; do
  set -- $cfg
  touch paper_2212_05159_b200/csrc/gcn.cu paper_2212_05159_b200/csrc/spgemm.cu
  CSRK_NVCC_EXTRA="-DCSRK_GCN_MINB=$1 -DCSRK_W_MINB=$2" python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
  echo "GCN_MINB=$1 W_MINB=$2"
  python bench.py --workload gcn --steps 5 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print({k:v['ms'] for k,v in d['ops'].items()})"
  python bench.py --workload cfg4 --steps 2 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print({k:v['ms'] for k,v in d['ops'].items() if 'gemm' in k})"
done
