"""Wall time of threshold calibration: the GPU select_thresholds (every
candidate of a layer replayed at once, one stream per candidate) vs the
reference's own select_thresholds on the host (one candidate after the other,
one core), on the same sequences and dense references.

  python tools/bench_calibration.py [--height 240 --width 320 --frames 6 --seqs 2 --steps 16]

Needs oracle/_ref (the reference build) for the CPU arm and the references.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_1808_05488_b200 import cbi  # noqa: E402
from tests import oracle  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--height", type=int, default=240)
ap.add_argument("--width", type=int, default=320)
ap.add_argument("--frames", type=int, default=6)
ap.add_argument("--seqs", type=int, default=2)
ap.add_argument("--steps", type=int, default=16)
ap.add_argument("--no-cpu", action="store_true")
a = ap.parse_args()

spec = cbi.make_seg_spec(1, a.height, a.width)
taus0 = [0.0] * 5
ref = oracle.RefNet(spec, taus0)
seqs = []
for q in range(a.seqs):
    f = cbi.gen_synthetic(cbi.SyntheticConfig(a.height, a.width, 3, a.frames, 4, 24, 3, 3, 0.004, 500 + q))
    seqs.append(cbi.EvalSequence(f, np.stack([ref.dense_forward(x) for x in f])))
cfg = cbi.CalibConfig(initial_tau=0.005, growth_factor=1.4, per_layer_budget=1e-3, max_steps=a.steps)
net = cbi.convert_to_cb(spec, taus0)
cbi.select_thresholds(net, seqs[:1], cbi.CalibConfig(max_steps=2))  # warm-up (graphs, allocations)
t0 = time.perf_counter()
got = cbi.select_thresholds(net, seqs, cfg)
gpu_s = time.perf_counter() - t0
out = {"workload": f"seg net {a.width}x{a.height}, {a.seqs} sequences x {a.frames} frames, max_steps {a.steps}",
       "gpu_seconds": gpu_s, "gpu_taus": got.taus, "replays": len(got.trace) + 5}
if not a.no_cpu:
    t0 = time.perf_counter()
    want = ref.select_thresholds(seqs, cfg)
    cpu_s = time.perf_counter() - t0
    out.update({"cpu_reference_seconds_1core": cpu_s, "cpu_taus": want.taus, "same_taus": got.taus == want.taus,
                "speedup": cpu_s / gpu_s})
print(json.dumps(out))
