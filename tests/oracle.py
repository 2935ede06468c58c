"""Test-side access to the CPU oracle (TEST INFRASTRUCTURE ONLY).

Two oracles, both built by oracle/Makefile (via __graft_entry__.build()):
  * ``Ref``  — the UNMODIFIED reference (cbi) compiled from /root/reference
    sources into oracle/_ref/libcbi_ref.so, driven through oracle/ref_shim.cpp.
  * ``Port`` — the plain-C restatement oracle/cbi_oracle.c
    (oracle/_build/liboracle.so), pinned bit-for-bit against ``Ref``.
Both are fed the same cbg_* description structs as the product, so every
parity test hands identical inputs to the GPU path and to the checker.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from paper_1808_05488_b200 import _lib
from paper_1808_05488_b200 import cbi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libcbi_ref.so")
PORT_SO = os.path.join(ROOT, "oracle", "_build", "liboracle.so")
REF_BENCH = os.path.join(ROOT, "oracle", "_ref", "ref_bench")

_vp = C.c_void_p
_ref = None
_port = None


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def port_available() -> bool:
    return os.path.exists(PORT_SO)


def _check(lib, prefix, st):
    if st != 0:
        msg = getattr(lib, prefix + "last_error")().decode()
        raise {1: cbi.InvalidInputError, 2: cbi.ConfigError}.get(st, RuntimeError)(msg)


def ref():
    global _ref
    if _ref is None:
        lib = C.CDLL(REF_SO)
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_net_create.argtypes = [C.POINTER(_lib.NetworkSpecC), _vp, C.c_int, _vp, C.c_int, C.POINTER(_vp)]
        lib.ref_net_destroy.argtypes = [_vp]
        lib.ref_net_clone.argtypes = [_vp, C.POINTER(_vp)]
        lib.ref_net_node_count.argtypes = [_vp]
        lib.ref_net_node_shape.argtypes = [_vp, C.c_int] + [C.POINTER(C.c_int)] * 4
        lib.ref_net_forward.argtypes = [_vp, _vp, C.c_int]
        lib.ref_net_reset.argtypes = [_vp]
        lib.ref_net_set_thresholds.argtypes = [_vp, _vp, C.c_int]
        lib.ref_net_read_output.argtypes = [_vp, C.c_int, _vp]
        lib.ref_net_read_state.argtypes = [_vp, C.c_int, _vp]
        lib.ref_net_read_stats.argtypes = [_vp, C.c_int] + [C.POINTER(C.c_int64)] * 3 + [_vp, _vp]
        lib.ref_dense_forward_row.argtypes = [_vp, _vp, C.c_int, _vp]
        lib.ref_select_thresholds.argtypes = [_vp, C.POINTER(_lib.EvalSequenceC), C.c_int,
                                              C.POINTER(_lib.CalibConfigC), _vp, _vp,
                                              C.POINTER(_lib.CalibTracePointC), C.c_int, C.POINTER(C.c_int)]
        lib.ref_sweep_threshold_factor.argtypes = [_vp, _vp, C.c_int, _vp, C.c_int, C.POINTER(_lib.EvalSequenceC),
                                                   C.c_int, C.c_int, C.POINTER(_lib.TradeoffRowC)]
        lib.ref_conv_create.argtypes = [C.POINTER(_lib.ConvSpecC), C.c_float, C.c_int, C.c_int, C.c_int, C.c_int,
                                        C.c_int, C.POINTER(_vp)]
        lib.ref_conv_destroy.argtypes = [_vp]
        lib.ref_conv_dims.argtypes = [_vp, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        lib.ref_conv_forward.argtypes = [_vp, _vp, _vp, _vp, C.c_int64, C.c_uint, C.POINTER(C.c_int64)]
        lib.ref_conv_read_output.argtypes = [_vp, _vp]
        lib.ref_conv_read_state.argtypes = [_vp, _vp]
        lib.ref_conv_read_changes.argtypes = [_vp, _vp, _vp, C.POINTER(C.c_int64)]
        lib.ref_conv_read_worst_case.argtypes = [_vp, _vp, C.POINTER(C.c_int64)]
        lib.ref_conv_set_tau.argtypes = [_vp, C.c_float]
        lib.ref_pool_create.argtypes = [C.c_int] * 7 + [C.POINTER(_vp)]
        lib.ref_pool_destroy.argtypes = [_vp]
        lib.ref_pool_forward.argtypes = [_vp, _vp, _vp, _vp, C.c_int64, C.c_int]
        lib.ref_pool_read_output.argtypes = [_vp, _vp]
        lib.ref_pool_read_changes.argtypes = [_vp, _vp, _vp, C.POINTER(C.c_int64)]
        lib.ref_gen_synthetic.argtypes = [C.POINTER(_lib.SyntheticConfigC), _vp, _vp]
        lib.ref_fill_random_weights.argtypes = [C.POINTER(_lib.NetworkSpecC), C.c_uint32, C.POINTER(_vp),
                                                C.POINTER(_vp)]
        lib.ref_detect_changes.argtypes = [_vp, _vp, C.c_int, C.c_int, C.c_int, C.c_float, C.c_int, _vp]
        lib.ref_dilate_window.argtypes = [_vp] + [C.c_int] * 8 + [_vp]
        lib.ref_propagate_changes.argtypes = [_vp, C.c_int, C.c_int, C.POINTER(_lib.ConvSpecC), _vp,
                                              C.POINTER(C.c_int), C.POINTER(C.c_int)]
        lib.ref_extract_indexes.argtypes = [_vp, C.c_int, C.c_int, _vp, C.POINTER(C.c_int64)]
        lib.ref_conv2d_dense.argtypes = [_vp, C.c_int, C.c_int, C.c_int, C.POINTER(_lib.ConvSpecC), _vp]
        lib.ref_im2col.argtypes = [_vp, C.c_int, C.c_int, C.c_int, C.POINTER(_lib.ConvSpecC), _vp, C.c_int64, _vp]
        lib.ref_gemm.argtypes = [C.POINTER(_lib.ConvSpecC), _vp, C.c_int64, _vp]
        lib.ref_maxpool_to.argtypes = [_vp] + [C.c_int] * 7 + [_vp]
        _ref = lib
    return _ref


def port():
    global _port
    if _port is None:
        lib = C.CDLL(PORT_SO)
        lib.cbo_last_error.restype = C.c_char_p
        lib.cbo_detect_changes.argtypes = [_vp, _vp, C.c_int, C.c_int, C.c_int, C.c_float, C.c_int, _vp]
        lib.cbo_dilate_window.argtypes = [_vp] + [C.c_int] * 8 + [_vp]
        lib.cbo_propagate_changes.argtypes = [_vp, C.c_int, C.c_int, C.POINTER(_lib.ConvSpecC), _vp,
                                              C.POINTER(C.c_int), C.POINTER(C.c_int)]
        lib.cbo_extract_indexes.argtypes = [_vp, C.c_int, C.c_int, _vp, C.POINTER(C.c_int64)]
        lib.cbo_im2col.argtypes = [_vp, C.c_int, C.c_int, C.c_int, C.POINTER(_lib.ConvSpecC), _vp, C.c_int64, _vp]
        lib.cbo_gemm.argtypes = [C.POINTER(_lib.ConvSpecC), _vp, C.c_int64, _vp]
        lib.cbo_update_output.argtypes = [_vp, C.c_int, C.c_int, C.c_int, _vp, _vp, C.c_int64, _vp, C.c_int]
        lib.cbo_conv2d_dense.argtypes = [_vp, C.c_int, C.c_int, C.c_int, C.POINTER(_lib.ConvSpecC), _vp]
        lib.cbo_maxpool_to.argtypes = [_vp] + [C.c_int] * 7 + [_vp]
        lib.cbo_net_create.argtypes = [C.POINTER(_lib.NetworkSpecC), _vp, C.c_int, _vp, C.c_int, C.POINTER(_vp)]
        lib.cbo_net_destroy.argtypes = [_vp]
        lib.cbo_net_node_count.argtypes = [_vp]
        lib.cbo_net_node_shape.argtypes = [_vp, C.c_int] + [C.POINTER(C.c_int)] * 4
        lib.cbo_net_forward.argtypes = [_vp, _vp]
        lib.cbo_net_reset.argtypes = [_vp]
        lib.cbo_net_set_thresholds.argtypes = [_vp, _vp, C.c_int]
        lib.cbo_net_read_output.argtypes = [_vp, C.c_int, _vp]
        lib.cbo_net_read_state.argtypes = [_vp, C.c_int, _vp]
        lib.cbo_net_read_changes.argtypes = [_vp, C.c_int, _vp, _vp, C.POINTER(C.c_int64)]
        _port = lib
    return _port


def f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def p(a):
    return None if a is None else a.ctypes.data_as(_vp)


# ---------------------------------------------------------------------------
# networks
# ---------------------------------------------------------------------------
class _NetBase:
    def _shapes(self, count_fn, shape_fn):
        self.shapes = []
        for i in range(count_fn(self.h)):
            k, c, hh, ww = C.c_int(), C.c_int(), C.c_int(), C.c_int()
            shape_fn(self.h, i, C.byref(k), C.byref(c), C.byref(hh), C.byref(ww))
            self.shapes.append((k.value, c.value, hh.value, ww.value))


class RefNet(_NetBase):
    """The reference CBNetwork (network.hpp:141-173) + its DenseNetwork."""

    def __init__(self, spec: cbi.NetworkSpec, taus, policies=None, mode=cbi.DetectMode.ClosedLoop):
        lib = ref()
        keep: list = []
        cs = spec._c(keep)
        t = f32(taus)
        pol = None if policies is None else np.ascontiguousarray([int(x) for x in policies], np.int32)
        h = _vp()
        _check(lib, "ref_", lib.ref_net_create(C.byref(cs), p(t), len(t), p(pol), int(mode), C.byref(h)))
        self.h = h
        self.lib = lib
        self.spec = spec
        self._shapes(lib.ref_net_node_count, lib.ref_net_node_shape)

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.ref_net_destroy(self.h)

    def clone(self):
        c = object.__new__(RefNet)
        h = _vp()
        _check(self.lib, "ref_", self.lib.ref_net_clone(self.h, C.byref(h)))
        c.h, c.lib, c.spec, c.shapes = h, self.lib, self.spec, list(self.shapes)
        return c

    def forward(self, frame, record_worst_case=False):
        _check(self.lib, "ref_", self.lib.ref_net_forward(self.h, p(f32(frame)), int(record_worst_case)))
        return self.output(-1)

    def output(self, node=-1):
        _, c, h, w = self.shapes[node]
        y = np.empty((c, h, w), np.float32)
        self.lib.ref_net_read_output(self.h, node, p(y))
        return y

    def state(self, node, shape=None):
        y = np.empty(shape if shape is not None else self.in_shape(node), np.float32)
        self.lib.ref_net_read_state(self.h, node, p(y))
        return y

    def in_shape(self, node):
        return None  # filled by callers that know the topology

    def stats(self, node):
        _, c, h, w = self.shapes[node]
        ch, eo, pr = C.c_int64(), C.c_int64(), C.c_int64()
        m = np.zeros((h, w), np.uint8)
        wc = np.zeros((h, w), np.uint8)
        self.lib.ref_net_read_stats(self.h, node, C.byref(ch), C.byref(eo), C.byref(pr), p(m), p(wc))
        return dict(changed_px=ch.value, eff_ops=eo.value, propagated_px=pr.value, map=m, worst_case_map=wc)

    def reset(self):
        self.lib.ref_net_reset(self.h)

    def set_thresholds(self, taus):
        t = f32(taus)
        _check(self.lib, "ref_", self.lib.ref_net_set_thresholds(self.h, p(t), len(t)))

    def select_thresholds(self, sequences, cfg):
        """The reference's select_thresholds (calibration.cpp:95-141) on this net."""
        keep: list = []
        seqs = cbi._sequences_c(list(sequences), keep)
        ov = np.ascontiguousarray(cfg.budget_overrides, dtype=np.float64)
        c = _lib.CalibConfigC(cfg.initial_tau, cfg.growth_factor, cfg.per_layer_budget,
                              ov.ctypes.data if len(ov) else None, len(ov), int(cfg.metric), int(cfg.aggregation),
                              cfg.max_steps)
        n_conv = sum(1 for d in self.spec.layers if d.kind == cbi.LayerKind.Conv)
        taus = np.zeros(n_conv, np.float32)
        cap = np.zeros(n_conv, np.uint8)
        ncap = max(1, n_conv * cfg.max_steps)
        trace = (_lib.CalibTracePointC * ncap)()
        n = C.c_int(0)
        _check(self.lib, "ref_", self.lib.ref_select_thresholds(self.h, seqs, len(sequences), C.byref(c), p(taus),
                                                                 cap.ctypes.data, trace, ncap, C.byref(n)))
        return cbi.CalibResult([float(t) for t in taus], [bool(x) for x in cap],
                               [cbi.CalibTracePoint(trace[i].layer, trace[i].tau, trace[i].loss)
                                for i in range(min(n.value, ncap))])

    def sweep_threshold_factor(self, base_tau, factors, sequences, metric=cbi.LossMetric.Mse):
        keep: list = []
        seqs = cbi._sequences_c(list(sequences), keep)
        bt = f32(base_tau)
        fa = np.ascontiguousarray(factors, np.float64)
        rows = (_lib.TradeoffRowC * max(1, len(fa)))()
        _check(self.lib, "ref_", self.lib.ref_sweep_threshold_factor(self.h, p(bt), len(bt), fa.ctypes.data, len(fa),
                                                                      seqs, len(sequences), int(metric), rows))
        return [cbi.TradeoffRow(rows[i].factor, rows[i].loss, rows[i].total_eff_ops, rows[i].wall_ns)
                for i in range(len(fa))]

    def dense_forward(self, frame, row=-1):
        """DenseNetwork::forward_all(frame)[row] (row indexes the spec, Act rows included)."""
        spec = self.spec
        if row < 0:
            row = len(spec.layers) + row
        shp = _row_shapes(spec)[row]
        y = np.empty(shp, np.float32)
        _check(self.lib, "ref_", self.lib.ref_dense_forward_row(self.h, p(f32(frame)), row, p(y)))
        return y


def _row_shapes(spec: cbi.NetworkSpec):
    shapes = []
    names = {}
    for i, d in enumerate(spec.layers):
        if d.from_:
            ins = [(-1 if s == "input" else names[s]) for s in d.from_]
        else:
            ins = [i - 1]
        src = [(spec.in_channels, spec.in_height, spec.in_width) if j < 0 else shapes[j] for j in ins]
        c, h, w = src[0]
        if d.kind == cbi.LayerKind.Conv:
            shp = (d.conv.out_channels, d.conv.output_height(h), d.conv.output_width(w))
        elif d.kind == cbi.LayerKind.Pool:
            oh = d.pool_out_h if d.pool_out_h > 0 else (h - d.pool_size) // d.pool_stride + 1
            ow = d.pool_out_w if d.pool_out_w > 0 else (w - d.pool_size) // d.pool_stride + 1
            shp = (c, oh, ow)
        elif d.kind == cbi.LayerKind.Concat:
            shp = (sum(s[0] for s in src), h, w)
        elif d.kind == cbi.LayerKind.Upsample:
            shp = (c, d.pool_out_h or h * d.upsample, d.pool_out_w or w * d.upsample)
        else:
            shp = (c, h, w)
        shapes.append(shp)
        if d.name:
            names[d.name] = i
    return shapes


class PortNet(_NetBase):
    """The plain-C restatement of the same network (oracle/cbi_oracle.c)."""

    def __init__(self, spec: cbi.NetworkSpec, taus, policies=None, mode=cbi.DetectMode.ClosedLoop):
        lib = port()
        keep: list = []
        cs = spec._c(keep)
        t = f32(taus)
        pol = None if policies is None else np.ascontiguousarray([int(x) for x in policies], np.int32)
        h = _vp()
        _check(lib, "cbo_", lib.cbo_net_create(C.byref(cs), p(t), len(t), p(pol), int(mode), C.byref(h)))
        self.h, self.lib = h, lib
        self._shapes(lib.cbo_net_node_count, lib.cbo_net_node_shape)

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.cbo_net_destroy(self.h)

    def forward(self, frame):
        _check(self.lib, "cbo_", self.lib.cbo_net_forward(self.h, p(f32(frame))))
        return self.output(-1)

    def output(self, node=-1):
        _, c, h, w = self.shapes[node]
        y = np.empty((c, h, w), np.float32)
        self.lib.cbo_net_read_output(self.h, node, p(y))
        return y

    def changes(self, node):
        _, c, h, w = self.shapes[node]
        m = np.zeros((h, w), np.uint8)
        rc = np.zeros((h * w, 2), np.int32)
        n = C.c_int64()
        self.lib.cbo_net_read_changes(self.h, node, p(m), p(rc), C.byref(n))
        return m, rc[:n.value].copy()

    def reset(self):
        self.lib.cbo_net_reset(self.h)

    def set_thresholds(self, taus):
        t = f32(taus)
        _check(self.lib, "cbo_", self.lib.cbo_net_set_thresholds(self.h, p(t), len(t)))


# ---------------------------------------------------------------------------
# layers
# ---------------------------------------------------------------------------
class RefConv:
    """The reference CBConvLayer (layers.hpp:45-69)."""

    def __init__(self, spec: cbi.ConvSpec, tau, policy=cbi.DetectionPolicy.Detect, fuse_relu=False,
                 mode=cbi.DetectMode.ClosedLoop, in_h=0, in_w=0):
        lib = ref()
        keep: list = []
        cs = spec._c(keep)
        h = _vp()
        _check(lib, "ref_", lib.ref_conv_create(C.byref(cs), float(tau), int(policy), int(fuse_relu), int(mode),
                                                in_h, in_w, C.byref(h)))
        self.h, self.lib, self.spec = h, lib, spec
        oh, ow = C.c_int(), C.c_int()
        lib.ref_conv_dims(h, C.byref(oh), C.byref(ow))
        self.out_h, self.out_w, self.in_h, self.in_w = oh.value, ow.value, in_h, in_w

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.ref_conv_destroy(self.h)

    def forward(self, x, up_map=None, up_idx=None, force=False, worst=False):
        m = None if up_map is None else np.ascontiguousarray(up_map, np.uint8)
        idx = None if up_idx is None else np.ascontiguousarray(np.asarray(up_idx, np.int32).reshape(-1, 2))
        eff = C.c_int64()
        flags = (1 if force else 0) | (2 if worst else 0)
        _check(self.lib, "ref_", self.lib.ref_conv_forward(self.h, p(f32(x)), p(m), p(idx),
                                                           0 if idx is None else len(idx), flags, C.byref(eff)))
        return eff.value

    @property
    def prev_output(self):
        y = np.empty((self.spec.out_channels, self.out_h, self.out_w), np.float32)
        self.lib.ref_conv_read_output(self.h, p(y))
        return y

    @property
    def state(self):
        y = np.empty((self.spec.in_channels, self.in_h, self.in_w), np.float32)
        self.lib.ref_conv_read_state(self.h, p(y))
        return y

    def changes(self):
        m = np.zeros((self.out_h, self.out_w), np.uint8)
        rc = np.zeros((self.out_h * self.out_w, 2), np.int32)
        n = C.c_int64()
        self.lib.ref_conv_read_changes(self.h, p(m), p(rc), C.byref(n))
        return m, rc[:n.value].copy()

    def worst_case(self):
        m = np.zeros((self.out_h, self.out_w), np.uint8)
        n = C.c_int64()
        self.lib.ref_conv_read_worst_case(self.h, p(m), C.byref(n))
        return m, n.value

    def set_tau(self, t):
        self.lib.ref_conv_set_tau(self.h, float(t))


class RefPool:
    def __init__(self, size, stride, channels, in_h, in_w, out_h, out_w):
        lib = ref()
        h = _vp()
        _check(lib, "ref_", lib.ref_pool_create(size, stride, channels, in_h, in_w, out_h, out_w, C.byref(h)))
        self.h, self.lib = h, lib
        self.channels, self.out_h, self.out_w = channels, out_h, out_w

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.ref_pool_destroy(self.h)

    def forward(self, x, up_map=None, up_idx=None, force=False):
        m = None if up_map is None else np.ascontiguousarray(up_map, np.uint8)
        idx = None if up_idx is None else np.ascontiguousarray(np.asarray(up_idx, np.int32).reshape(-1, 2))
        _check(self.lib, "ref_", self.lib.ref_pool_forward(self.h, p(f32(x)), p(m), p(idx),
                                                           0 if idx is None else len(idx), int(force)))

    @property
    def prev_output(self):
        y = np.empty((self.channels, self.out_h, self.out_w), np.float32)
        self.lib.ref_pool_read_output(self.h, p(y))
        return y

    def changes(self):
        m = np.zeros((self.out_h, self.out_w), np.uint8)
        rc = np.zeros((self.out_h * self.out_w, 2), np.int32)
        n = C.c_int64()
        self.lib.ref_pool_read_changes(self.h, p(m), p(rc), C.byref(n))
        return m, rc[:n.value].copy()


# ---------------------------------------------------------------------------
# generators (reference harness)
# ---------------------------------------------------------------------------
def ref_gen_synthetic(cfg: cbi.SyntheticConfig, with_corners=False):
    c = _lib.SyntheticConfigC(cfg.height, cfg.width, cfg.channels, cfg.n_frames, cfg.n_objects, cfg.object_size,
                              cfg.velocity_y, cfg.velocity_x, cfg.noise_std, cfg.seed)
    frames = np.empty((cfg.n_frames, cfg.channels, cfg.height, cfg.width), np.float32)
    corners = np.empty((cfg.n_frames, max(cfg.n_objects, 0), 2), np.int32) if with_corners else None
    _check(ref(), "ref_", ref().ref_gen_synthetic(C.byref(c), p(frames), p(corners)))
    return (frames, corners) if with_corners else frames


def ref_fill_random_weights(spec: cbi.NetworkSpec, seed: int):
    """Reference fill_random_weights; returns [(weights, bias)] per conv row."""
    convs = [d for d in spec.layers if d.kind == cbi.LayerKind.Conv]
    outs = [(np.zeros(d.conv.weight_count(), np.float32), np.zeros(d.conv.out_channels, np.float32)) for d in convs]
    for d in convs:  # struct needs placeholder buffers of the right size
        if d.conv.weights is None:
            d.conv.weights = np.zeros(d.conv.weight_count(), np.float32)
            d.conv.bias = np.zeros(d.conv.out_channels, np.float32)
    keep: list = []
    cs = spec._c(keep)
    W = (_vp * max(1, len(outs)))(*[w.ctypes.data for w, _ in outs])
    B = (_vp * max(1, len(outs)))(*[b.ctypes.data for _, b in outs])
    _check(ref(), "ref_", ref().ref_fill_random_weights(C.byref(cs), seed, W, B))
    return outs


# ---------------------------------------------------------------------------
# metrics (reference tests/oracles.hpp:59-66)
# ---------------------------------------------------------------------------
REF_STATS_CSV = os.path.join(os.path.dirname(REF_SO), "ref_stats_csv")


def ref_seg_stats_csv(seed, height, width, taus, synth: "cbi.SyntheticConfig", with_reference=False) -> str:
    """The reference's forward_sequence + write_stats_csv (timing off) for the
    seg net (make_seg7_spec layers at derived dims, fill_random_weights(seed)) on
    gen_synthetic(synth), run by oracle/_ref/ref_stats_csv."""
    import subprocess
    c = synth
    args = [REF_STATS_CSV, str(seed), str(height), str(width)] + [repr(float(t)) for t in taus] + [
        str(c.n_frames), str(c.n_objects), str(c.object_size), str(c.velocity_y), str(c.velocity_x),
        repr(float(c.noise_std)), str(c.seed), "1" if with_reference else "0"]
    return subprocess.run(args, capture_output=True, text=True, check=True).stdout


# observed max_rel_err per test (tests/conftest.py writes it to $CBG_PARITY_OUT:
# the measured maxima behind every tolerance in the GPU tests)
OBSERVED: dict = {}


def dense_forward64(spec: cbi.NetworkSpec, frame):
    """Float64 dense evaluation of a layer manifest in numpy, an independent
    formulation (no im2col, no fp32 rounding) used to pin the oracle's EXTENSIONS
    (leaky ReLU, upsampling) that the reference cannot check. Returns every row's
    output, Act rows included."""
    outs = []
    names = {}
    x0 = np.asarray(frame, np.float64)
    for i, d in enumerate(spec.layers):
        ins = [(-1 if s == "input" else names[s]) for s in d.from_] if d.from_ else [i - 1]
        src = [x0 if j < 0 else outs[j] for j in ins]
        x = src[0]
        if d.kind == cbi.LayerKind.Conv:
            cv = d.conv
            c, h, w = x.shape
            oh, ow = cv.output_height(h), cv.output_width(w)
            xp = np.zeros((c, h + 2 * cv.padding + cv.kernel_h, w + 2 * cv.padding + cv.kernel_w))
            xp[:, cv.padding:cv.padding + h, cv.padding:cv.padding + w] = x
            wt = np.asarray(cv.weights, np.float64).reshape(cv.out_channels, c, cv.kernel_h, cv.kernel_w)
            y = np.zeros((cv.out_channels, oh, ow))
            for kj in range(cv.kernel_h):
                for ki in range(cv.kernel_w):
                    patch = xp[:, kj:kj + (oh - 1) * cv.stride + 1:cv.stride, ki:ki + (ow - 1) * cv.stride + 1:cv.stride]
                    y += np.einsum("oc,chw->ohw", wt[:, :, kj, ki], patch)
            y += np.asarray(cv.bias, np.float64)[:, None, None]
            if d.fuse_relu:
                y = np.where(y < 0, y * d.act_slope, y)
        elif d.kind == cbi.LayerKind.Act:
            y = np.where(x < 0, x * d.act_slope, x)
        elif d.kind == cbi.LayerKind.Pool:
            c, h, w = x.shape
            oh = d.pool_out_h if d.pool_out_h > 0 else (h - d.pool_size) // d.pool_stride + 1
            ow = d.pool_out_w if d.pool_out_w > 0 else (w - d.pool_size) // d.pool_stride + 1
            y = np.full((c, oh, ow), -np.inf)
            for kj in range(d.pool_size):
                for ki in range(d.pool_size):
                    for jo in range(oh):
                        j = jo * d.pool_stride + kj
                        if j >= h:
                            continue
                        cols = np.arange(ow) * d.pool_stride + ki
                        ok = cols < w
                        y[:, jo, ok] = np.maximum(y[:, jo, ok], x[:, j, cols[ok]])
        elif d.kind == cbi.LayerKind.Upsample:
            y = x.repeat(d.upsample, axis=1).repeat(d.upsample, axis=2)
            y = y[:, :d.pool_out_h or y.shape[1], :d.pool_out_w or y.shape[2]]
        elif d.kind == cbi.LayerKind.Concat:
            y = np.concatenate(src, axis=0)
        else:  # Add
            y = sum(src)
        outs.append(y)
        if d.name:
            names[d.name] = i
    return outs


def max_rel_err(a, b) -> float:
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if a.size == 0:
        return 0.0
    e = float(np.max(np.abs(a - b) / np.maximum(1.0, np.abs(b))))
    test = os.environ.get("PYTEST_CURRENT_TEST", "").split(" ")[0]
    if test:
        OBSERVED[test] = max(OBSERVED.get(test, 0.0), e)
    return e
