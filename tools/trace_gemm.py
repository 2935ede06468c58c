"""Per-K-block pipeline timeline of the GEMM kernel (CTA 0), instrumented build.

  make -C paper_1808_05488_b200/csrc trace
  CBG_LIB=libcbg_trace.so python tools/trace_gemm.py --cin 16 --cout 64 --k 7 --h 237 --w 317
"""
import argparse
import ctypes as C
import os
import sys

os.environ.setdefault("CBG_LIB", "libcbg_trace.so")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1808_05488_b200 import _lib, cbi  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cin", type=int, default=16)
ap.add_argument("--cout", type=int, default=64)
ap.add_argument("--k", type=int, default=7)
ap.add_argument("--h", type=int, default=237)
ap.add_argument("--w", type=int, default=317)
a = ap.parse_args()
rng = np.random.default_rng(0)
spec = cbi.ConvSpec(a.cin, a.cout, a.k, a.k, 1, a.k // 2)
spec.weights = rng.uniform(-0.1, 0.1, spec.weight_count()).astype(np.float32)
spec.bias = np.zeros(a.cout, np.float32)
layer = cbi.CBConvLayer(spec, 0.0, in_height=a.h, in_width=a.w)
x = rng.uniform(0, 1, (a.cin, a.h, a.w)).astype(np.float32)
for _ in range(3):
    layer.forward(x, force_full_update=True)
buf = np.zeros((6, 4096), np.uint64)
n = _lib.lib.cbg_debug_gemm_trace(buf.ctypes.data_as(C.c_void_p), buf.size)
assert n > 0, "not an instrumented build"
names = ["fetch_issued", "conv_saw_raw", "mma_saw_full", "mma_issued", "fetch_got_empty", "conv_done"]
valid = np.where(buf[3] > 0)[0]
g = valid[valid > 0]
t0 = buf[4, 0]
print("K-blocks traced:", len(valid))
for ev in range(6):
    print(f"{names[ev]:>16}", ((buf[ev, g[:12]].astype(np.int64) - int(t0))).tolist())
def d(e1, e2):
    return (buf[e2, g].astype(np.int64) - buf[e1, g].astype(np.int64))
print("median cycles: got_empty->issued %d, issued->raw %d, raw->conv_done %d, conv_done->full %d, full->mma_issued %d"
      % tuple(int(np.median(d(*p))) for p in ((4, 0), (0, 1), (1, 5), (5, 2), (2, 3))))
step = np.diff(buf[3, g].astype(np.int64))
print("median cycles between consecutive MMA K-blocks:", int(np.median(step)), " mean:", int(step.mean()))
