#!/bin/bash
# A/B of the SpMM paths on config 2 (ops report of bench.py, 10 steps); variants as arguments
cd "$(dirname "$0")/.."
for v in "$@"; do
  env $v python bench.py --steps 10 --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2>gpurun_out/ab.err || tail -3 gpurun_out/ab.err
  python -c "
import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1])
print('$v', d['ms_per_step'], {k:v['ms'] for k,v in d['ops'].items() if 'spm' in k}, d['gate']['spmm_fwd_bwd'])"
done
