#!/bin/bash
# ncu launch list + DRAM traffic of one steady-state frame (-> profiles/ncu_traffic.json on the box and
# gpurun_out/), then the default bench and the cfg5 bench
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --print-units base --csv --log-file gpurun_out/traffic.csv python tools/profile_run.py --streams 64 --frames 6 \
  --labels gpurun_out/labels.json > gpurun_out/profile_run.log 2>&1
python tools/ncu_traffic.py gpurun_out/traffic.csv --streams 64 --labels gpurun_out/labels.json --out gpurun_out/ncu_traffic.json > /dev/null && cp gpurun_out/ncu_traffic.json profiles/ncu_traffic.json
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_cfg2.log 2> gpurun_out/bench_cfg2.err
timeout 900 python bench.py --config cfg5 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg5.log 2> gpurun_out/bench_cfg5.err
tail -2 gpurun_out/bench_cfg2.err gpurun_out/bench_cfg5.err
