#!/bin/bash
# round-end evidence: the frame traffic list (copied to profiles/ncu_traffic.json,
# which bench.py reads for roofline.traffic), the bench line (default flags), the
# cfg5 line, the ncu launch list of the bench command, full captures of the top kernels
set -x
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --print-units base --csv --log-file gpurun_out/traffic.csv python tools/profile_run.py --streams 64 --frames 6 \
  --labels gpurun_out/labels.json > gpurun_out/profile_run.log 2>&1
python tools/ncu_traffic.py gpurun_out/traffic.csv --streams 64 --labels gpurun_out/labels.json --out gpurun_out/ncu_traffic.json > /dev/null \
  && cp gpurun_out/ncu_traffic.json profiles/ncu_traffic.json
timeout 900 python bench.py > gpurun_out/bench_cfg2.log 2> gpurun_out/bench_cfg2.err
timeout 900 python bench.py --config cfg5 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg5.log 2> gpurun_out/bench_cfg5.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --print-units base --csv \
  --log-file gpurun_out/ncu_launches_bench.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline \
  --profile-steps 1 --dense-steps 2 --sweep-steps 0 --no-e2e > gpurun_out/ncu_bench.log 2>&1
bash tools/ncu_kernel.sh conv_gemm_kernel 10 g256f
bash tools/ncu_kernel.sh conv_gemm_kernel 9 g64f
bash tools/ncu_kernel.sh dilate_compact 25 dcl1f
