#!/usr/bin/env python3
"""Full-size parity report (test infrastructure): the GPU stream set against
the unmodified reference (oracle/_ref) on the BASELINE configs at the sizes
whose throughput bench.py / tools/bench_configs.py report, plus the fp64
anchor (tests/fullsize.py). Writes profiles/r02_parity.json.

  python tools/parity_report.py [--only cfg2,cfg5] [--out profiles/r02_parity.json]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1808_05488_b200 import cbi  # noqa: E402
from tests import fullsize  # noqa: E402


def pnm_seq(h, w, n, objects, size, vy, vx, noise, seed):
    raw = cbi.gen_synthetic(cbi.SyntheticConfig(h, w, 3, n, objects, size, vy, vx, noise, seed))
    return cbi.from_pnm8(cbi.to_pnm8(raw))


def configs():
    # cfg2: the bench workload (bench.py defaults: 640x480, 6 objects x 40 px,
    # v=4, 8-bit frames, tau 0.05), streams 0 and 1 of the bench's seeds
    yield ("cfg2", "scene-labeling net 640x480, bench workload (streams 1000, 1001), 6 frames",
           cbi.make_seg_spec(1, 480, 640), [0.05] * 5,
           [pnm_seq(480, 640, 6, 6, 40, 4, 4, 0.0, 1000 + s) for s in range(2)], 6)
    # cfg3: OpenPose-style, full width, 2 stages, 368x368 (tools/bench_configs.py)
    sp = cbi.make_openpose_spec(5, 368, 368, width_div=1, stages=2)
    nc = sum(1 for d in sp.layers if d.kind == cbi.LayerKind.Conv)
    yield ("cfg3", "OpenPose-style full width, 2 stages, 368x368, 1 moving subject", sp, [0.02] * nc,
           [pnm_seq(368, 368, 3, 1, 64, 5, 3, 0.0, 31 + s) for s in range(2)], 3)
    # cfg4: tiny-YOLO-style, full width, 1920x1080
    sp = cbi.make_yolo_spec(9, 1080, 1920)
    nc = sum(1 for d in sp.layers if d.kind == cbi.LayerKind.Conv)
    yield ("cfg4", "tiny-YOLO-style full width 1920x1080, 3 objects + sensor noise", sp, [0.03] * nc,
           [pnm_seq(1080, 1920, 3, 3, 48, 4, 6, 0.002, 77 + s) for s in range(2)], 3)
    # cfg5: the scene-labeling net at 1080p (the multi-GPU config's per-stream work)
    yield ("cfg5", "scene-labeling net 1920x1080 (cfg5 streams 1000, 1001)", cbi.make_seg_spec(1, 1080, 1920),
           [0.05] * 5, [pnm_seq(1080, 1920, 3, 6, 40, 4, 4, 0.0, 1000 + s) for s in range(2)], 3)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_parity.json"))
    a = ap.parse_args()
    only = set(x for x in a.only.split(",") if x)
    out = {}
    if os.path.exists(a.out):
        with open(a.out) as fh:
            out = json.load(fh)
    for name, desc, spec, taus, streams, n in configs():
        if only and name not in only:
            continue
        t0 = time.time()
        rep = fullsize.run_parity(spec, taus, streams, n, anchor_frames=(0, -1),
                                  log=lambda m: print(f"[{name} {time.time() - t0:.0f}s] {m}", flush=True))
        out[name] = {"workload": desc, "summary": fullsize.summary(rep), "per_frame": rep["per_frame"],
                     "wall_s": round(time.time() - t0, 1)}
        print(name, json.dumps(out[name]["summary"]), flush=True)
        with open(a.out, "w") as fh:
            json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
