set -x
for F in 1 0; do
CBG_FUSE_POOL=$F timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --print-units base --csv --log-file gpurun_out/traffic_f$F.csv python tools/profile_run.py --streams 64 --frames 6 --labels gpurun_out/labels_f$F.json > gpurun_out/pr_f$F.log 2>&1
python tools/ncu_traffic.py gpurun_out/traffic_f$F.csv --streams 64 --labels gpurun_out/labels_f$F.json --out gpurun_out/ncu_traffic_f$F.json > /dev/null
done
python - <<'PY'
import json
for F in (1, 0):
    d = json.load(open(f"gpurun_out/ncu_traffic_f{F}.json"))
    print("fuse", F, "total us", round(sum(d["duration_us"].values()), 1))
    for k, v in d["duration_us"].items(): print(f"  {k:14s} {v:8.1f} us {d['dram_bytes_per_launch'][k]/1e6:8.2f} MB")
PY
