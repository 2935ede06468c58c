#!/bin/bash
# ncu launch-list durations per kernel label for several environment settings of
# one build:  tools/ncu_env_ab.sh "CBG_X=0" "CBG_X=1" ...   (profile_run.py, 64 streams, last frame)
i=0
for E in "$@"; do
  env $E timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --print-units base --csv --log-file gpurun_out/eab_$i.csv python tools/profile_run.py --streams 64 --frames 6 --labels gpurun_out/eab_labels_$i.json > /dev/null 2>&1
  python tools/ncu_traffic.py gpurun_out/eab_$i.csv --streams 64 --labels gpurun_out/eab_labels_$i.json --out gpurun_out/eab_$i.json > /dev/null
  i=$((i+1))
done
python - "$@" <<'PY'
import json, sys
ds = [json.load(open(f"gpurun_out/eab_{i}.json"))["duration_us"] for i in range(len(sys.argv) - 1)]
labels = list(dict.fromkeys(k for d in ds for k in d))
print(f"{'kernel':14s}" + "".join(f"{E[:18]:>20s}" for E in sys.argv[1:]))
for k in labels:
    print(f"{k:14s}" + "".join(f"{d.get(k, 0):20.1f}" for d in ds))
print(f"{'total':14s}" + "".join(f"{sum(d.values()):20.1f}" for d in ds))
PY
