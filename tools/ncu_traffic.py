"""Turn an ncu CSV of one steady-state frame (tools/profile_run.py, one stream
set of S streams) into profiles/ncu_traffic.json: DRAM bytes and duration per
kernel label ("<node>.<kernel>", the labels bench.py's roofline uses).

  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none --print-units base --csv --log-file gpurun_out/traffic.csv \
      python tools/profile_run.py --streams 64 --frames 6 --labels gpurun_out/labels.json
  python tools/ncu_traffic.py gpurun_out/traffic.csv --streams 64 --labels gpurun_out/labels.json
"""
import argparse
import csv
import json
import os


ap = argparse.ArgumentParser()
ap.add_argument("csv")
ap.add_argument("--labels", required=True, help="labels.json written by tools/profile_run.py --labels")
ap.add_argument("--streams", type=int, required=True)
ap.add_argument("--height", type=int, default=480)
ap.add_argument("--width", type=int, default=640)
ap.add_argument("--out", default=os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                              "profiles", "ncu_traffic.json"))
a = ap.parse_args()
rows = list(csv.reader(open(a.csv)))
hdr = None
launches = {}
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        lid = int(d["ID"])
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "")
        v *= {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1e3, "msecond": 1e6}.get(unit, 1.0)
        launches.setdefault(lid, {"name": d["Kernel Name"]})[d["Metric Name"]] = v
LABELS = json.load(open(a.labels))
ids = sorted(launches)
frame = [launches[i] for i in ids[-len(LABELS):]]  # the last frame
assert "begin_frame" in frame[0]["name"], frame[0]["name"]
out = {"streams": a.streams, "height": a.height, "width": a.width,
       "source": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                 "(--clock-control none) over tools/profile_run.py, last of 6 frames",
       "dram_bytes_per_launch": {}, "duration_us": {}}
for lab, l in zip(LABELS, frame):
    out["dram_bytes_per_launch"][lab] = l.get("dram__bytes_read.sum", 0) + l.get("dram__bytes_write.sum", 0)
    out["duration_us"][lab] = l.get("gpu__time_duration.sum", 0) / 1000.0
json.dump(out, open(a.out, "w"), indent=1)
print(json.dumps(out, indent=1))
