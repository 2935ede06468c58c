#!/bin/bash
# A/B of library builds on the bench workload: [N=rounds] tools/ab.sh libA.so libB.so ...
N=${N:-3}
for i in $(seq $N); do
  for L in "$@"; do
    CBG_LIB=$L timeout 300 python bench.py --sweep-steps 0 --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/ab.json')); k={n: v['us'] for n, v in d['roofline']['all_kernels'].items()}; print('$L', round(d['value']), round(d['ms_per_step'],4), {n: k[n] for n in ('L5.gemm','L3.gemm','L6.gemm') if n in k}, 'dilcomp', round(sum(v for n, v in k.items() if n.endswith('dilcomp')), 1))"
  done
done
