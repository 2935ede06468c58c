#!/bin/bash
# bench A/B over environment settings of one build: [N=rounds] tools/env_ab.sh "CBG_X=0" "CBG_X=1"
N=${N:-2}
for i in $(seq $N); do for E in "$@"; do
  env $E timeout 300 python bench.py --sweep-steps 0 --no-cpu-baseline --no-e2e --dense-steps 0 > gpurun_out/ab.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ab.json')); k={n: v['us'] for n, v in d['roofline']['all_kernels'].items()}; print('$E', round(d['value']), round(d['ms_per_step'],4), 'dilcomp', round(sum(v for n, v in k.items() if n.endswith('dilcomp')), 1))"
done; done
