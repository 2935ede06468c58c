"""Kernel timeline of the bench workload (4 stream groups, device-resident 8-bit
frames) from CUPTI via torch.profiler: which kernels of which group run when,
and how much of a step the GPU spends with 0 / 1 / 2+ kernels in flight.

  python tools/timeline.py [--steps 4] [--persistent-sms -1] > gpurun_out/timeline.txt
"""
import argparse
import collections
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1808_05488_b200 import cbi  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=4)
ap.add_argument("--groups", type=int, default=4)
ap.add_argument("--streams", type=int, default=64)
ap.add_argument("--persistent-sms", type=int, default=-1)
ap.add_argument("--json", default="")
a = ap.parse_args()
torch.cuda.set_device(0)
S, G, H, W = a.streams, a.groups, 480, 640
Sg = S // G
n_sm = torch.cuda.get_device_properties(0).multi_processor_count
psms = a.persistent_sms if a.persistent_sms >= 0 else (-(-n_sm // 3) if G >= 3 else -(-n_sm // G))
ctxs = [cbi.Context(0) for _ in range(G)]
for c in ctxs:
    c.set_persistent_sms(psms)
spec = cbi.make_seg_spec(1, H, W)
L = 8
h8 = np.stack([cbi.to_pnm8(cbi.gen_synthetic(cbi.SyntheticConfig(H, W, 3, L, 6, 40, 4, 4, 0.0, 1000 + s)))
               for s in range(S)], axis=1)
dev8 = torch.from_numpy(np.ascontiguousarray(h8)).cuda()
nets = [cbi.convert_to_cb(spec, [0.05] * 5, n_streams=Sg, ctx=ctxs[g]) for g in range(G)]
labels = nets[0].kernel_labels()
order = list(range(1, L)) + list(range(L - 2, 1, -1))
for k in range(8):
    for g in range(G):
        nets[g].enqueue_device_u8(dev8[0 if k == 0 else order[k % len(order)], g * Sg].data_ptr())
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for k in range(a.steps):
        for g in range(G):
            nets[g].enqueue_device_u8(dev8[order[(8 + k) % len(order)], g * Sg].data_ptr())
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ks = []
for e in ev:
    ks.append((e.time_range.start, e.time_range.end, e.name, getattr(e, "device_resource_id", 0)))
ks.sort()
t0, t1 = ks[0][0], max(k[1] for k in ks)
span = t1 - t0
# short kernel names
def short(n):
    for key in ("conv_gemm_kernel<256", "conv_gemm_kernel<64", "conv_exact_kernel<16", "conv_exact_kernel<8",
                "detect_frame_s8", "detect_list", "dilate_compact", "pool_kernel", "begin_frame", "detect_frame"):
        if key in n:
            return key
    return n[:30]
busy = collections.defaultdict(float)
for s_, e_, n, r in ks:
    busy[short(n)] += e_ - s_
# concurrency histogram
pts = sorted([(s_, 1) for s_, _, _, _ in ks] + [(e_, -1) for _, e_, _, _ in ks])
hist = collections.defaultdict(float)
cur, last = 0, pts[0][0]
for t, d in pts:
    hist[min(cur, 4)] += t - last
    cur += d
    last = t
print(f"steps {a.steps}, groups {G}, persistent SMs {psms}; span {span:.0f} us = {span / a.steps:.0f} us per step "
      f"({S * a.steps / span * 1e6:.0f} frames/s under the profiler)")
print("time with n kernels in flight:", {k: f"{100 * v / span:.1f}%" for k, v in sorted(hist.items())})
print("kernel busy time per step (sum over launches, us):")
for n, v in sorted(busy.items(), key=lambda x: -x[1]):
    print(f"  {n:28s} {v / a.steps:8.1f}")
# GEMM concurrency: time with k GEMMs in flight
gp = sorted([(s_, 1) for s_, _, n, _ in ks if "conv_gemm" in n] + [(e_, -1) for _, e_, n, _ in ks if "conv_gemm" in n])
gh = collections.defaultdict(float)
cur, last = 0, t0
for t, d in gp:
    gh[cur] += t - last
    cur += d
    last = t
gh[0] += t1 - last
print("time with k tensor GEMMs in flight:", {k: f"{100 * v / span:.1f}%" for k, v in sorted(gh.items())})
if a.json:
    json.dump([{"start": s_ - t0, "end": e_ - t0, "name": short(n), "stream": r} for s_, e_, n, r in ks],
              open(a.json, "w"))
