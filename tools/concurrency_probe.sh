#!/bin/bash
# Bench throughput vs stream groups / streams (is more concurrency the lever? DESIGN.md §8.28),
# then an ncu --set full of the last frame's deep compactions.

for cfg in "--groups 4 --streams 64" "--groups 8 --streams 128" "--groups 4 --streams 128" "--groups 8 --streams 64"; do
  timeout 300 python bench.py --sweep-steps 0 --no-cpu-baseline --no-e2e --dense-steps 0 --profile-steps 1 --steps 30 $cfg 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', round(d['value']), d['ms_per_step'], d['clocks'].get('sm_mhz'))"
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:dilate_compact -s 27 -c 3 -f -o gpurun_out/dc_deep python tools/profile_run.py --streams 64 > gpurun_out/dc_deep.log 2>&1; tail -2 gpurun_out/dc_deep.log
