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
buf = np.zeros(6 * 4096 + 4 * 160 + 7 * 64, np.uint64)
_lib.lib.cbg_debug_gemm_trace(buf.ctypes.data_as(C.c_void_p), buf.size)
cta = buf[6 * 4096:6 * 4096 + 640].reshape(4, 160)[:, :148].astype(np.int64)
epi = buf[6 * 4096 + 640:6 * 4096 + 640 + 192].reshape(3, 64).astype(np.int64)
chk = buf[6 * 4096 + 640 + 192:].reshape(4, 64).astype(np.int64)
t0 = cta[0].min()
rel = (cta - t0) / 1000.0
print("changed px per stream (traced layer):", net.counts()[-1].tolist()[:16])
print("start   us: min %.1f med %.1f max %.1f" % (rel[0].min(), np.median(rel[0]), rel[0].max()))
print("setup   us: min %.1f med %.1f max %.1f" % (rel[1].min(), np.median(rel[1]), rel[1].max()))
print("mma end us: min %.1f med %.1f max %.1f" % (rel[2].min(), np.median(rel[2]), rel[2].max()))
print("end     us: min %.1f med %.1f max %.1f" % (rel[3].min(), np.median(rel[3]), rel[3].max()))
print("epilogue tail (end - mma end) median us: %.1f" % np.median(rel[3] - rel[2]))

# CTA 0's K-block pipeline in this steady-state launch: only the first n_kb
# entries belong to it (older launches left the rest)
node = net.nodes()[-1]
cout, cin = node.out_shape[0], node.in_shape[0]
k = int(round((node.ops_per_pixel / (2 * cout * cin)) ** 0.5))
KB = (k * k * ((cin + 3) // 4 * 4) + 31) // 32
tiles = [(int(c) + 127) // 128 for c in net.counts()[-1]]
n_tiles = sum(tiles) * ((cout + 3) // 4 * 4 + 255) // 256
n_kb = len(range(0, sum(tiles), 148)) * KB
tr = buf[:6 * 4096].reshape(6, 4096)[:, :min(n_kb, 4096)].astype(np.int64)


def d(e1, e2):
    return tr[e2, 1:] - tr[e1, 1:]


print("CTA 0: %d K-blocks (KB=%d)  median cycles: got_empty->issued %d, issued->raw %d, raw->conv_done %d, "
      "conv_done->full %d, full->mma_issued %d" % ((tr.shape[1], KB) + tuple(
          int(np.median(d(*p))) for p in ((4, 0), (0, 1), (1, 5), (5, 2), (2, 3)))))
step = np.diff(tr[3])
span = tr[3, -1] - tr[3, 0]
print("MMA K-block period: median %d mean %.0f cycles; %d gaps > 4x median hold %.1f%% of the span" % (
    int(np.median(step)), step.mean(), int((step > 4 * np.median(step)).sum()),
    100.0 * step[step > 4 * np.median(step)].sum() / max(1, span)))
ns = (cta[2, 0] - cta[1, 0])
print("CTA 0: %d MMA cycles over %.1f us of globaltimer -> %.2f GHz effective SM clock" % (span, ns / 1e3,
                                                                                        span / max(1, ns)))

nt0 = len(range(0, sum(tiles), 148))
e = epi[:, :nt0]
print("CTA 0 epilogue per tile (cycles): tfull->TMEM released", (e[1] - e[0]).tolist())
print("                                  released->stores done", (e[2] - e[1]).tolist())
print("  MMA idle at tile boundaries: tfull(t) -> next K-block issue:",
      [int(tr[2, KB * (t + 1)] - e[0, t]) if KB * (t + 1) < tr.shape[1] else -1 for t in range(nt0 - 1)])
nch = (cout + 3) // 4 * 4 // 32 if cout >= 32 else 1
c = chk[:, :min(64, nt0 * nch)]
print("epilogue chunks (cycles): TMEM ld+wait", (c[1] - c[0]).tolist()[:16])
print("                          compute+stage ", (c[2] - c[1]).tolist()[:16])
print("                          stores        ", (c[3] - c[2]).tolist()[:16])
if len(sys.argv) > 3 and sys.argv[3] == "window":
    names = ["issued", "conv_saw_raw", "mma_saw_full", "mma_issued", "fetch_got_empty", "conv_done"]
    lo = min(100, tr.shape[1] - 20)
    base = int(tr[4, lo])
    print("K-block window (cycles relative to fetch_got_empty of block %d):" % lo)
    print("  kb " + " ".join(f"{n:>15s}" for n in names))
    for kb in range(lo, lo + 16):
        print(f"{kb:4d} " + " ".join(f"{int(tr[e, kb]) - base:15d}" for e in range(6)))
