"""Repro: low-change sequences through a multi-stream set (debug helper)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1808_05488_b200 import cbi
S = int(sys.argv[1]) if len(sys.argv) > 1 else 16
ob, sz = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (1, 8)
H, W = 480, 640
spec = cbi.make_seg_spec(1, H, W)
frames = np.stack([cbi.gen_synthetic(cbi.SyntheticConfig(H, W, 3, 6, ob, sz, 4, 4, 0.0, 1000 + s))
                   for s in range(S)], axis=1)
net = cbi.convert_to_cb(spec, [0.05] * 5, n_streams=S)
for t in range(6):
    net.enqueue(np.ascontiguousarray(frames[t]))
    net.synchronize()
    print(t, net.counts()[:, :4].tolist(), flush=True)
