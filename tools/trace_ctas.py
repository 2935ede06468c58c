"""Per-CTA timeline (globaltimer) of the L5 GEMM launch inside the seg net, instrumented build.

  CBG_LIB=libcbg_trace.so python tools/trace_ctas.py
"""
import ctypes as C
import os
import sys

os.environ.setdefault("CBG_LIB", "libcbg_trace.so")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1808_05488_b200 import _lib, cbi  # noqa: E402

S, H, W = int(sys.argv[1]) if len(sys.argv) > 1 else 64, 480, 640
spec = cbi.make_seg_spec(1, H, W)
# truncated so the last GEMM launch of a frame is the traced layer (L5 default; "L3" / "L6")
upto = {"L3": 4, "L5": 7, "L6": 8}[sys.argv[2] if len(sys.argv) > 2 else "L5"]
spec.layers = spec.layers[:upto]
frames = np.stack([cbi.gen_synthetic(cbi.SyntheticConfig(H, W, 3, 6, 6, 40, 4, 4, 0.0, 1000 + s)) for s in range(S)],
                  axis=1)
n_conv = sum(1 for d in spec.layers if d.kind == cbi.LayerKind.Conv)
net = cbi.convert_to_cb(spec, [0.05] * n_conv, n_streams=S)
for t in range(6):
    net.enqueue(np.ascontiguousarray(frames[t]))
net.synchronize()
buf = np.zeros(6 * 4096 + 4 * 160, np.uint64)
_lib.lib.cbg_debug_gemm_trace(buf.ctypes.data_as(C.c_void_p), buf.size)
cta = buf[6 * 4096:].reshape(4, 160)[:, :148].astype(np.int64)
t0 = cta[0].min()
rel = (cta - t0) / 1000.0
print("changed px per stream (traced layer):", net.counts()[-1].tolist()[:16])
print("start   us: min %.1f med %.1f max %.1f" % (rel[0].min(), np.median(rel[0]), rel[0].max()))
print("setup   us: min %.1f med %.1f max %.1f" % (rel[1].min(), np.median(rel[1]), rel[1].max()))
print("mma end us: min %.1f med %.1f max %.1f" % (rel[2].min(), np.median(rel[2]), rel[2].max()))
print("end     us: min %.1f med %.1f max %.1f" % (rel[3].min(), np.median(rel[3]), rel[3].max()))
print("epilogue tail (end - mma end) median us: %.1f" % np.median(rel[3] - rel[2]))

# CTA 0's K-block pipeline in this steady-state launch
tr = buf[:6 * 4096].reshape(6, 4096)
valid = np.where(tr[3] > 0)[0]
g = valid[valid > 0]


def d(e1, e2):
    return tr[e2, g].astype(np.int64) - tr[e1, g].astype(np.int64)


print("CTA 0 K-blocks:", len(valid), " median cycles: got_empty->issued %d, issued->raw %d, raw->conv_done %d, "
      "conv_done->full %d, full->mma_issued %d" % tuple(int(np.median(d(*p))) for p in ((4, 0), (0, 1), (1, 5), (5, 2),
                                                                                       (2, 3))))
step = np.diff(tr[3, valid].astype(np.int64))
print("MMA K-block period: median %d mean %d; gaps > 3000 cycles: %d (sum %d cycles of %d)" % (
    int(np.median(step)), int(step.mean()), int((step > 3000).sum()), int(step[step > 3000].sum()), int(step.sum())))
