#!/bin/bash
# cfg4 SpGEMM op times under build variants: tools/ab_cfg4.sh "<nvcc extra flags>" ...
cd "$(dirname "$0")/.."
for v in "$@"; do
  CSRK_NVCC_EXTRA="$v" python -c "from paper_2212_05159_b200 import build; build.build(force=True)" > gpurun_out/b.log 2>&1 || tail -5 gpurun_out/b.log
  python bench.py --workload cfg4 --steps 3 > gpurun_out/ab4.json 2> gpurun_out/ab4.err || tail -3 gpurun_out/ab4.err
  python -c "
import json;d=json.loads(open('gpurun_out/ab4.json').read().strip().splitlines()[-1])
print('[$v]', round(d['ms_per_step'],1), {k:v['ms'] for k,v in d['ops'].items()})"
done
