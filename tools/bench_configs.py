"""Throughput of the other BASELINE.json configs (bench.py measures configs[1]).

  python tools/bench_configs.py [--only cfg1,cfg3,cfg4,cfg5] > gpurun_out/configs.jsonl

One JSON line per measurement: frames/s of the change-based path (frames
resident in HBM, CUDA events around K steps after W warm-up steps, every
stream of the set per step), the same kernels' dense path, and the measured
changed-pixel fraction of the first layer. Frames are 8-bit PNM-quantized
gen_synthetic sequences played ping-pong (as in bench.py).

  cfg1  single CBconv 3x3 16->32 on 64x64, ~5% changed output pixels (the
        reference's CPU-runnable case; 1024 streams per launch)
  cfg3  OpenPose-style pose net (make_openpose_spec, full width, 2 stages) at
        368x368, one moving subject
  cfg4  tiny-YOLO-style detector (make_yolo_spec, full width, ReLU) at 1920x1080,
        change-rate sweep 0.1-100%
  cfg4v3  tiny-YOLOv3-style detector (make_yolov3_spec: leaky ReLU, x2 upsample +
        concat route, two heads; the extensions the reference lacks) at
        1920x1080, change-rate sweep 0.1-100%
  cfg5  scene-labeling net at 1920x1080, 64 streams on one GPU (the N=1 point
        of the 64-stream scaling config)
"""
import argparse
import json
import os
import sys
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1808_05488_b200 import cbi  # noqa: E402


def frames_for(S, H, W, R, objects, size, vel, noise, seed0=1000, C=3):
    out = torch.empty((R, S, C, H, W), dtype=torch.float32, pin_memory=True)
    o = out.numpy()

    def one(s):
        raw = cbi.gen_synthetic(cbi.SyntheticConfig(H, W, C, R, objects, size, vel, vel, noise, seed0 + s))
        o[:, s] = cbi.from_pnm8(cbi.to_pnm8(raw)) if C == 3 else raw
    with ThreadPoolExecutor(max_workers=min(16, os.cpu_count() or 1)) as pool:
        list(pool.map(one, range(S)))
    return out.cuda()


def timed(net, dev, steps, warmup, dense=False):
    R = dev.shape[0]
    order = list(range(1, R)) + list(range(R - 2, 0, -1))
    net.set_dense(dense)
    net.enqueue_device(dev[0].data_ptr())
    for k in range(warmup):
        net.enqueue_device(dev[order[k % len(order)]].data_ptr())
    net.synchronize()
    ext = torch.cuda.ExternalStream(net.ctx.stream)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(ext)
    for k in range(steps):
        net.enqueue_device(dev[order[(warmup + k) % len(order)]].data_ptr())
    t1.record(ext)
    t1.synchronize()
    counts = net.counts()
    return t0.elapsed_time(t1) / steps, counts


def measure(name, spec, taus, dev, steps, warmup, extra):
    S = dev.shape[1]
    net = cbi.convert_to_cb(spec, taus, n_streams=S)
    ms, counts = timed(net, dev, steps, warmup)
    n0 = net.nodes()[0]
    l1 = float(counts[0].mean()) / (n0.out_shape[1] * n0.out_shape[2])
    dms, _ = timed(net, dev, max(2, steps // 4), 1, dense=True)
    ops = sum(n.ops_per_pixel * n.out_shape[1] * n.out_shape[2] for n in net.nodes()
              if n.kind == cbi.LayerKind.Conv)
    line = {"config": name, "streams": S, "height": spec.in_height, "width": spec.in_width,
            "frames_per_s": S / (ms / 1000.0), "ms_per_step": ms,
            "dense_frames_per_s": S / (dms / 1000.0), "speedup_vs_dense": dms / ms,
            "l1_changed_pct": 100.0 * l1, "dense_gflop_per_frame": ops / 1e9}
    line.update(extra)
    print(json.dumps(line), flush=True)
    del net


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="cfg1,cfg3,cfg4,cfg4v3,cfg5")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    a = ap.parse_args()
    want = set(a.only.split(","))
    torch.cuda.set_device(0)

    if "cfg1" in want:
        S, H, W = 1024, 64, 64
        spec = cbi.NetworkSpec(16, H, W, [cbi.LayerDesc(cbi.LayerKind.Conv, "cbconv",
                                                        conv=cbi.ConvSpec(16, 32, 3, 3, 1, 1))])
        cbi.fill_random_weights(spec, 1)
        # 16-channel frames: a static background with one 12x12 block redrawn per
        # frame (-> 14x14 = 4.8% of the output pixels change)
        rng = np.random.default_rng(7)
        base = rng.uniform(0, 1, (S, 16, H, W)).astype(np.float32)
        R = 6
        fr = np.repeat(base[None], R, axis=0)
        for t in range(R):
            y, x = rng.integers(0, H - 12, S), rng.integers(0, W - 12, S)
            for s in range(S):
                fr[t, s, :, y[s]:y[s] + 12, x[s]:x[s] + 12] = rng.uniform(0, 1, (16, 12, 12))
        dev = torch.from_numpy(fr).cuda()
        measure("cfg1 single CBconv 3x3 16->32, 64x64", spec, [0.05], dev, a.steps * 5, a.warmup,
                {"note": "one 12x12 block redrawn per frame"})
        del dev

    if "cfg3" in want:
        spec = cbi.make_openpose_spec(1, 368, 368, width_div=1, stages=2)
        n = sum(1 for d in spec.layers if d.kind == cbi.LayerKind.Conv)
        dev = frames_for(16, 368, 368, 6, 1, 96, 4, 0.0)
        measure("cfg3 OpenPose-style (VGG-19 front, 2 stages), 368x368", spec, [0.05] * n, dev, a.steps, a.warmup,
                {"synthetic": "1 moving subject (96 px, v=4)"})
        del dev

    for key, make, label in (("cfg4", cbi.make_yolo_spec, "cfg4 tiny-YOLO-style detector, 1920x1080"),
                             ("cfg4v3", cbi.make_yolov3_spec,
                              "cfg4 tiny-YOLOv3-style detector (leaky ReLU, upsample route), 1920x1080")):
        if key not in want:
            continue
        spec = make(1, 1080, 1920)
        n = sum(1 for d in spec.layers if d.kind == cbi.LayerKind.Conv)
        for pt in ((1, 16), (4, 32), (12, 64), (40, 96), (120, 128), "noise"):
            if pt == "noise":  # every pixel changes every frame: the change-based path's worst case
                gen = torch.Generator(device="cuda").manual_seed(99)
                dev = torch.randint(0, 256, (5, 8, 3, 1080, 1920), generator=gen, device="cuda",
                                    dtype=torch.uint8).float() / 255.0
                syn = "uniform noise every frame"
            else:
                dev = frames_for(8, 1080, 1920, 5, pt[0], pt[1], 4, 0.0)
                syn = f"{pt[0]} objects x {pt[1]} px, v=4"
            measure(label, spec, [0.05] * n, dev, a.steps, a.warmup, {"synthetic": syn})
            del dev
            torch.cuda.empty_cache()

    if "cfg5" in want:
        spec = cbi.make_seg_spec(1, 1080, 1920)
        dev = frames_for(64, 1080, 1920, 4, 12, 80, 4, 0.0)
        measure("cfg5 scene-labeling net, 64 x 1920x1080 streams on 1 GPU", spec, [0.05] * 5, dev, a.steps, a.warmup,
                {"synthetic": "12 objects x 80 px, v=4", "note": "the N=1 point of the 64-stream scaling config"})
        del dev


if __name__ == "__main__":
    main()
