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

S, H, W = 16, 480, 640
spec = cbi.make_seg_spec(1, H, W)
# the network without L6/L7 so the last GEMM launch of a frame is L5
spec.layers = spec.layers[:7]
frames = np.stack([cbi.gen_synthetic(cbi.SyntheticConfig(H, W, 3, 6, 6, 40, 4, 4, 0.0, 1000 + s)) for s in range(S)],
                  axis=1)
net = cbi.convert_to_cb(spec, [0.05] * 3, n_streams=S)
for t in range(6):
    net.enqueue(np.ascontiguousarray(frames[t]))
net.synchronize()
buf = np.zeros(6 * 4096 + 4 * 160, np.uint64)
_lib.lib.cbg_debug_gemm_trace(buf.ctypes.data_as(C.c_void_p), buf.size)
cta = buf[6 * 4096:].reshape(4, 160)[:, :148].astype(np.int64)
t0 = cta[0].min()
rel = (cta - t0) / 1000.0
print("L5 changed px per stream:", net.counts()[-1].tolist())
print("start   us: min %.1f med %.1f max %.1f" % (rel[0].min(), np.median(rel[0]), rel[0].max()))
print("setup   us: min %.1f med %.1f max %.1f" % (rel[1].min(), np.median(rel[1]), rel[1].max()))
print("mma end us: min %.1f med %.1f max %.1f" % (rel[2].min(), np.median(rel[2]), rel[2].max()))
print("end     us: min %.1f med %.1f max %.1f" % (rel[3].min(), np.median(rel[3]), rel[3].max()))
print("epilogue tail (end - mma end) median us: %.1f" % np.median(rel[3] - rel[2]))
