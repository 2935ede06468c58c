#!/bin/bash
# ncu launch-list durations per kernel label for several library builds:
#   tools/ncu_ab.sh libA.so libB.so ...   (profile_run.py, 64 streams, last frame)
for L in "$@"; do
  CBG_LIB=$L timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --print-units base --csv --log-file gpurun_out/ab_$L.csv python tools/profile_run.py --streams 64 --frames 6 --labels gpurun_out/ab_labels_$L.json > /dev/null 2>&1
  python tools/ncu_traffic.py gpurun_out/ab_$L.csv --streams 64 --labels gpurun_out/ab_labels_$L.json --out gpurun_out/ab_$L.json > /dev/null
done
python - "$@" <<'PY'
import json, sys
ds = [json.load(open(f"gpurun_out/ab_{L}.json"))["duration_us"] for L in sys.argv[1:]]
labels = list(ds[0])
print(f"{'kernel':14s}" + "".join(f"{L[:18]:>20s}" for L in sys.argv[1:]))
for k in labels:
    print(f"{k:14s}" + "".join(f"{d.get(k, 0):20.1f}" for d in ds))
print(f"{'total':14s}" + "".join(f"{sum(d.values()):20.1f}" for d in ds))
PY
