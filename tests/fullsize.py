"""Full-size network parity against the reference (TEST INFRASTRUCTURE ONLY).

Runs a CBNetwork stream set on the GPU beside one unmodified reference
CBNetwork per stream (oracle/_ref, one host thread each: ctypes releases the
GIL) on identical gen_synthetic sequences and reports, per frame and node:
  * change-map agreement and changed_px equality (bit-exact at
    layer 1, agreement reported for deeper layers),
  * max_rel_err of every node's retained output (tests/oracles.hpp:59-66),
  * an fp64 anchor per closed-loop Detect conv: with closed-loop detection a
    layer's retained output is act(conv(state)) at every pixel (acceptance C2,
    acceptance.cpp:102-123), so each side's output is compared with a
    double-accumulator convolution of ITS OWN state (the reference's
    conv2d_brute, tests/oracles.hpp:15-37, computed here with float64
    torch.conv2d). The GPU's error against fp64 is then bounded by a multiple
    of the reference's own error against fp64: an error budget that does not
    depend on where the two sides' masks happen to agree.
"""
from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor

import numpy as np

from paper_1808_05488_b200 import cbi
from tests import oracle


def conv_fp64(x: np.ndarray, conv: cbi.ConvSpec, relu: bool, device=None) -> np.ndarray:
    """act(conv2d(x) + b) with float64 products and sums (conv2d_brute)."""
    import torch
    import torch.nn.functional as F
    dev = device or ("cuda" if torch.cuda.is_available() else "cpu")
    c, h, w = x.shape
    oh, ow = conv.output_height(h), conv.output_width(w)
    xt = torch.from_numpy(np.ascontiguousarray(x)).to(dev, torch.float64)[None]
    # pinned output dims larger than the derived ones read zero padding
    need_h = (oh - 1) * conv.stride + conv.kernel_h - 2 * conv.padding
    need_w = (ow - 1) * conv.stride + conv.kernel_w - 2 * conv.padding
    xt = F.pad(xt, (0, max(0, need_w - w), 0, max(0, need_h - h)))
    wt = torch.from_numpy(np.asarray(conv.weights, np.float32).reshape(
        conv.out_channels, conv.in_channels, conv.kernel_h, conv.kernel_w)).to(dev, torch.float64)
    bt = torch.from_numpy(np.asarray(conv.bias, np.float32)).to(dev, torch.float64)
    y = F.conv2d(xt, wt, bt, stride=conv.stride, padding=conv.padding)[0, :, :oh, :ow]
    if relu:
        y = torch.clamp(y, min=0.0)
    return y.cpu().numpy()


def rel_err64(a: np.ndarray, ref64: np.ndarray) -> float:
    """max_rel_err of a float32 tensor against a float64 one (oracles.hpp:59-66)."""
    a = np.asarray(a, np.float64)
    return float(np.max(np.abs(a - ref64) / np.maximum(1.0, np.abs(ref64)))) if a.size else 0.0


def conv_rows(spec: cbi.NetworkSpec):
    """node name -> ConvSpec of the spec row (Act rows are absorbed into nodes)."""
    out = {}
    for i, d in enumerate(spec.layers):
        if d.kind == cbi.LayerKind.Conv:
            out[d.name or f"L{i + 1}"] = d.conv
    return out


def run_parity(spec, taus, streams, n_frames, anchor_frames=(-1,), anchor_streams=(0,), log=None):
    """streams: list of [n_frames, C, H, W] sequences (one per camera stream).
    Returns a report dict (JSON-serialisable)."""
    S = len(streams)
    net = cbi.convert_to_cb(spec, taus, n_streams=S)
    refs = [oracle.RefNet(spec, taus) for _ in range(S)]
    nodes = net.nodes()
    rows = conv_rows(spec)
    anchor_frames = {f % n_frames for f in anchor_frames}
    rep = {"streams": S, "frames": n_frames, "nodes": [n.name for n in nodes], "per_frame": []}
    with ThreadPoolExecutor(max_workers=S) as pool:
        for t in range(n_frames):
            batch = np.stack([streams[s][t] for s in range(S)]).astype(np.float32)
            net.enqueue(batch)
            list(pool.map(lambda s: refs[s].forward(streams[s][t]), range(S)))
            counts = net.counts()
            fr = {"frame": t, "l1_bit_exact": True, "agree": {}, "changed_px_equal": {}, "changed_px": {},
                  "max_rel_err": {}, "final_max_rel_err": 0.0, "anchor": {}}
            for i, n in enumerate(nodes):
                ag, eq, err = [], [], []
                for s in range(S):
                    st = refs[s].stats(i)
                    gm, gi = net.node_changes(i, s)
                    if i == 0:
                        ok = np.array_equal(gm, st["map"]) and np.array_equal(
                            gi, np.argwhere(st["map"]).astype(np.int32))
                        fr["l1_bit_exact"] = fr["l1_bit_exact"] and bool(ok)
                    ag.append(float(np.mean(gm == st["map"])))
                    eq.append(int(counts[i, s]) == st["changed_px"])
                    err.append(oracle.max_rel_err(net.node_output(i, s), refs[s].output(i)))
                fr["agree"][n.name] = min(ag)
                fr["changed_px_equal"][n.name] = all(eq)
                fr["changed_px"][n.name] = int(counts[i].sum())
                fr["max_rel_err"][n.name] = max(err)
            fr["final_max_rel_err"] = fr["max_rel_err"][nodes[-1].name]
            if t in anchor_frames:
                for i, n in enumerate(nodes):
                    if not (n.kind == cbi.LayerKind.Conv and n.policy == cbi.DetectionPolicy.Detect):
                        continue
                    eg = er = 0.0
                    for s in anchor_streams:
                        xs_g = net.node_state(i, s)
                        xs_r = refs[s].state(i, n.in_shape)
                        eg = max(eg, rel_err64(net.node_output(i, s), conv_fp64(xs_g, rows[n.name], n.fuse_relu)))
                        er = max(er, rel_err64(refs[s].output(i), conv_fp64(xs_r, rows[n.name], n.fuse_relu)))
                    fr["anchor"][n.name] = {"gpu_vs_fp64": eg, "ref_vs_fp64": er}
            rep["per_frame"].append(fr)
            if log:
                log(f"frame {t}: l1 exact {fr['l1_bit_exact']} min agree {min(fr['agree'].values()):.6f} "
                    f"final err {fr['final_max_rel_err']:.3g} anchor {fr['anchor']}")
    return rep


def summary(rep):
    """Worst values over the run: the numbers the tests assert and profiles/ records."""
    pf = rep["per_frame"]
    names = rep["nodes"]
    out = {"l1_bit_exact": all(f["l1_bit_exact"] for f in pf),
           "min_agree": {n: min(f["agree"][n] for f in pf) for n in names},
           "changed_px_equal": {n: all(f["changed_px_equal"][n] for f in pf) for n in names},
           "max_rel_err": {n: max(f["max_rel_err"][n] for f in pf) for n in names},
           "final_max_rel_err": max(f["final_max_rel_err"] for f in pf)}
    anc = {}
    for f in pf:
        for n, v in f["anchor"].items():
            a = anc.setdefault(n, {"gpu_vs_fp64": 0.0, "ref_vs_fp64": 0.0})
            a["gpu_vs_fp64"] = max(a["gpu_vs_fp64"], v["gpu_vs_fp64"])
            a["ref_vs_fp64"] = max(a["ref_vs_fp64"], v["ref_vs_fp64"])
    out["anchor"] = anc
    return out
