#!/bin/bash
# e2e A/B over an environment knob: tools/e2e_ab.sh VAR "v1 v2 ..." [rounds]
VAR=$1; VALS=$2; N=${3:-2}
for i in $(seq $N); do
  for v in $VALS; do
    env $VAR=$v timeout 400 python bench.py --sweep-steps 0 --no-cpu-baseline --dense-steps 0 --profile-steps 1 > gpurun_out/e2e_ab.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/e2e_ab.json')); print('$VAR=$v', 'value', round(d['value']), 'e2e', round(d['e2e']['value']), 'full', round(d['e2e_full_output']['value']), 'f32', round(d['e2e_f32']['value']) if d.get('e2e_f32') else None)"
  done
done
