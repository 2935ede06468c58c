"""Short steady-state run of the bench workload for ncu (no timing printed).

  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches.csv python tools/profile_run.py
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_1808_05488_b200 import cbi  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--streams", type=int, default=16)
ap.add_argument("--frames", type=int, default=6)
ap.add_argument("--height", type=int, default=480)
ap.add_argument("--width", type=int, default=640)
ap.add_argument("--objects", type=int, default=6)
ap.add_argument("--object-size", type=int, default=40)
ap.add_argument("--velocity", type=int, default=4)
ap.add_argument("--dense", action="store_true")
ap.add_argument("--ingest", choices=["u8", "f32"], default="u8", help="frame format, as bench.py --ingest")
ap.add_argument("--labels", default="", help="write the frame's kernel labels (launch order) here")
a = ap.parse_args()
S, H, W = a.streams, a.height, a.width
spec = cbi.make_seg_spec(1, H, W)
frames = np.stack([cbi.gen_synthetic(cbi.SyntheticConfig(H, W, 3, a.frames, a.objects, a.object_size, a.velocity,
                                                         a.velocity, 0.0, 1000 + s)) for s in range(S)], axis=1)
net = cbi.convert_to_cb(spec, [0.05] * 5, n_streams=S)
if a.dense:
    net.set_dense(True)
pnm = cbi.to_pnm8(frames)  # [T, S, H, W, C]: what bench.py feeds (u8), or its byte/255 (f32)
for t in range(a.frames):
    if a.ingest == "u8":
        net.enqueue_u8(np.ascontiguousarray(pnm[t]))
    else:
        net.enqueue(np.ascontiguousarray(cbi.from_pnm8(pnm[t])))
net.synchronize()
if a.labels:
    import json
    with open(a.labels, "w") as fh:
        json.dump(net.kernel_labels(), fh)
print("counts L1..L7 (stream 0):", net.counts()[:, 0].tolist())
