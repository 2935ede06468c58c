"""Numerical study for DESIGN.md §9.3: error of the 3xFP16 split vs fp16 main term + e4m3 correction
terms (kind::f8f6f4 would run them at twice the fp16 rate) on L5-like dot products (K = 64 x 49).
Exact products, fp64 sums: the split's own error only (the GPU adds fp32 accumulation, ~3e-5 at L5)."""
# numerical study: L5-like dot products (K = 64*49 = 3136), activations ReLU-like, He-uniform weights.
import numpy as np
rng = np.random.default_rng(0)
K, N, M = 3136, 64, 512
x = np.maximum(rng.standard_normal((M, K)).astype(np.float32), 0) * 0.5
w = (rng.uniform(-1, 1, (K, N)) * np.sqrt(6.0 / K)).astype(np.float32)
ref = x.astype(np.float64) @ w.astype(np.float64)

def split16(a, e):  # a * 2^-e = hi + lo in fp16 (round to nearest)
    s = (a.astype(np.float64) * 2.0**-e)
    hi = s.astype(np.float16)
    lo = (s - hi.astype(np.float64)).astype(np.float16)
    return hi, lo

def e4m3(a):  # round to e4m3 (3 mantissa bits, max 448), with a power-of-two scale chosen per tensor
    a = np.asarray(a, np.float64)
    amax = np.abs(a).max()
    sc = 2.0 ** np.floor(np.log2(448.0 / amax)) if amax > 0 else 1.0
    v = a * sc
    m, ex = np.frexp(v)               # v = m * 2^ex, |m| in [0.5,1)
    m = np.round(m * 16) / 16         # 4 significant bits (1 implicit + 3)
    q = np.ldexp(m, ex)
    q = np.where(np.abs(v) < 2.0**-9, 0.0, q)  # (subnormals ignored: coarse)
    return q / sc

ex = int(np.ceil(np.log2(np.abs(x).max()))) - 14
ew = int(np.ceil(np.log2(np.abs(w).max()))) - 14
xh, xl = split16(x, ex); wh, wl = split16(w, ew)
f = lambda a: a.astype(np.float64)
main = f(xh) @ f(wh)
corr16 = f(xh) @ f(wl) + f(xl) @ f(wh)
scale = 2.0 ** (ex + ew)
y3 = (main + corr16) * scale                     # 3xFP16 (exact products, fp64 sums: the split's own error)
corr8 = e4m3(f(xh)) @ e4m3(f(wl)) + e4m3(f(xl)) @ e4m3(f(wh))
y8 = (main + corr8) * scale                      # fp16 main + fp8 corrections
y1 = main * scale                                # 1xFP16 (no corrections)
den = np.abs(ref).max()
for name, y in (("3xFP16", y3), ("fp16 + fp8 corrections", y8), ("1xFP16", y1)):
    print(f"{name:24s} max|err|/max|y| = {np.abs(y - ref).max() / den:.2e}")
