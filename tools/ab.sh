#!/bin/bash
# A/B of two library builds on the bench workload: tools/ab.sh libA.so libB.so [rounds]
A=$1; B=$2; N=${3:-3}
for i in $(seq $N); do
  for L in $A $B; do
    CBG_LIB=$L timeout 300 python bench.py --sweep-steps 0 --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('$L', round(d['value']), round(d['ms_per_step'],4))"
  done
done
