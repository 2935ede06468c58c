"""CPU: pin the oracle.

1. The plain-C restatement (oracle/cbi_oracle.c) is bit-identical to the
   unmodified reference build (oracle/_ref) on random inputs, primitive by
   primitive and for whole networks.
2. Both reproduce the reference test suite's known-answer vectors
   (tests/golden/kats.json, each citing its reference test file:line).
3. The product's host-side harness (gen_synthetic / fill_random_weights inside
   libcbg) is byte-identical to the reference's (io.cpp:499-566), so GPU and
   CPU runs see the same frames and weights.
"""
import ctypes as C
import json
import os

import numpy as np
import pytest

from paper_1808_05488_b200 import _lib, cbi
from tests import oracle
from tests.oracle import p

HERE = os.path.dirname(os.path.abspath(__file__))
need_ref = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
need_port = pytest.mark.skipif(not oracle.port_available(), reason="oracle/_build not built")


def conv_spec(rng, cin, cout=None, k=None, stride=None, pad=None):
    k = k or int(rng.choice([1, 3, 5, 7]))
    s = cbi.ConvSpec(cin, cout or int(rng.integers(1, 9)), k, k, stride or int(rng.integers(1, 3)),
                     int(pad if pad is not None else rng.integers(0, k // 2 + 1)))
    s.weights = rng.uniform(-0.3, 0.3, s.weight_count()).astype(np.float32)
    s.bias = rng.uniform(-0.1, 0.1, s.out_channels).astype(np.float32)
    return s


# ---------------------------------------------------------------------------
# restatement == reference, primitive by primitive
# ---------------------------------------------------------------------------
@need_ref
@need_port
@pytest.mark.parametrize("seed", range(20))
def test_primitives_bit_identical(seed):
    rng = np.random.default_rng(seed)
    R, P = oracle.ref(), oracle.port()
    c, h, w = int(rng.integers(1, 6)), int(rng.integers(3, 14)), int(rng.integers(3, 14))
    x = rng.uniform(-1, 1, (c, h, w)).astype(np.float32)
    st = (x + rng.uniform(-0.2, 0.2, x.shape) * (rng.random(x.shape) < 0.3)).astype(np.float32)
    tau = float(rng.choice([0.0, 0.05, 0.1]))
    for mode in (0, 1):
        s1, s2 = st.copy(), st.copy()
        m1, m2 = np.zeros((h, w), np.uint8), np.zeros((h, w), np.uint8)
        assert R.ref_detect_changes(p(x), p(s1), c, h, w, tau, mode, p(m1)) == 0
        assert P.cbo_detect_changes(p(x), p(s2), c, h, w, tau, mode, p(m2)) == 0
        assert np.array_equal(m1, m2) and np.array_equal(s1, s2)
    spec = conv_spec(rng, c)
    try:
        oh, ow = spec.output_height(h), spec.output_width(w)
    except cbi.InvalidInputError:
        return
    keep = []
    cs = spec._c(keep)
    m = (rng.random((h, w)) < 0.2).astype(np.uint8)
    d1, d2 = np.zeros((oh, ow), np.uint8), np.zeros((oh, ow), np.uint8)
    R.ref_dilate_window(p(m), h, w, spec.kernel_h, spec.kernel_w, spec.stride, spec.padding, oh, ow, p(d1))
    P.cbo_dilate_window(p(m), h, w, spec.kernel_h, spec.kernel_w, spec.stride, spec.padding, oh, ow, p(d2))
    assert np.array_equal(d1, d2)
    n1, n2 = C.c_int64(), C.c_int64()
    rc1, rc2 = np.zeros((oh * ow, 2), np.int32), np.zeros((oh * ow, 2), np.int32)
    R.ref_extract_indexes(p(d1), oh, ow, p(rc1), C.byref(n1))
    P.cbo_extract_indexes(p(d2), oh, ow, p(rc2), C.byref(n2))
    assert n1.value == n2.value and np.array_equal(rc1, rc2)
    K = c * spec.kernel_h * spec.kernel_w
    n = n1.value
    col1, col2 = np.zeros((max(n, 1), K), np.float32), np.zeros((max(n, 1), K), np.float32)
    assert R.ref_im2col(p(x), c, h, w, C.byref(cs), p(rc1), n, p(col1)) == 0
    assert P.cbo_im2col(p(x), c, h, w, C.byref(cs), p(rc2), n, p(col2)) == 0
    assert np.array_equal(col1, col2)
    y1, y2 = np.zeros((spec.out_channels, max(n, 1)), np.float32), np.zeros((spec.out_channels, max(n, 1)),
                                                                            np.float32)
    R.ref_gemm(C.byref(cs), p(col1), n, p(y1))
    P.cbo_gemm(C.byref(cs), p(col2), n, p(y2))
    assert np.array_equal(y1[:, :n], y2[:, :n])  # exact: same non-FMA sequential order
    z1, z2 = np.zeros((spec.out_channels, oh, ow), np.float32), np.zeros((spec.out_channels, oh, ow), np.float32)
    R.ref_conv2d_dense(p(x), c, h, w, C.byref(cs), p(z1))
    P.cbo_conv2d_dense(p(x), c, h, w, C.byref(cs), p(z2))
    assert np.array_equal(z1, z2)
    if h >= 2 and w >= 2:
        ph, pw = (h - 2) // 2 + 1, (w - 2) // 2 + 1
        q1, q2 = np.zeros((c, ph, pw), np.float32), np.zeros((c, ph, pw), np.float32)
        R.ref_maxpool_to(p(x), c, h, w, 2, 2, ph, pw, p(q1))
        P.cbo_maxpool_to(p(x), c, h, w, 2, 2, ph, pw, p(q2))
        assert np.array_equal(q1, q2)


def random_net(rng, c, h, w, n_convs):
    """tests/oracles.hpp:104-147 analogue: random conv/pool chain, dims >= 4."""
    spec = cbi.NetworkSpec(c, h, w, [])
    for i in range(n_convs):
        s = conv_spec(rng, c)
        oh, ow = h + 2 * s.padding - s.kernel_h, w + 2 * s.padding - s.kernel_w
        if not (oh >= 0 and ow >= 0 and oh // s.stride + 1 >= 4 and ow // s.stride + 1 >= 4):
            s.stride, s.padding = 1, s.kernel_h // 2
        spec.layers.append(cbi.LayerDesc(cbi.LayerKind.Conv, f"conv{i}", [], s, bool(rng.integers(0, 2))))
        c, h, w = s.out_channels, s.output_height(h), s.output_width(w)
        if i + 1 < n_convs and h >= 8 and w >= 8 and rng.integers(0, 2):
            spec.layers.append(cbi.LayerDesc(cbi.LayerKind.Pool, f"pool{i}", pool_size=2, pool_stride=2))
            h, w = (h - 2) // 2 + 1, (w - 2) // 2 + 1
    return spec


@need_ref
@need_port
@pytest.mark.parametrize("seed", range(10))
def test_network_restatement_bit_identical(seed):
    rng = np.random.default_rng(1000 + seed)
    c, h, w = int(rng.integers(1, 4)), int(rng.integers(12, 33)), int(rng.integers(12, 33))
    spec = random_net(rng, c, h, w, int(rng.integers(2, 6)))
    nconv = sum(1 for d in spec.layers if d.kind == cbi.LayerKind.Conv)
    taus = [float(rng.choice([0.0, 0.02, 0.05])) for _ in range(nconv)]
    mode = cbi.DetectMode(int(rng.integers(0, 2)))
    r, q = oracle.RefNet(spec, taus, None, mode), oracle.PortNet(spec, taus, None, mode)
    x = rng.uniform(0, 1, (c, h, w)).astype(np.float32)
    for t in range(6):
        if t == 4:
            r.set_thresholds([v * 0.5 for v in taus])
            q.set_thresholds([v * 0.5 for v in taus])
        assert np.array_equal(r.forward(x), q.forward(x))
        for i in range(len(r.shapes)):
            assert np.array_equal(r.stats(i)["map"], q.changes(i)[0])
        x = x.copy()
        k = int(rng.integers(0, h * w // 6 + 1))
        x[:, rng.integers(0, h, k), rng.integers(0, w, k)] = rng.uniform(0, 1, (c, k)).astype(np.float32)


@need_ref
@need_port
def test_joins_restatement_bit_identical():
    """test_network.cpp:12-55 diamond with Add and Concat joins."""
    for join in (cbi.LayerKind.Add, cbi.LayerKind.Concat):
        rng = np.random.default_rng(50 + int(join))
        stem = conv_spec(rng, 2, k=3, stride=1, pad=1)
        spec = cbi.NetworkSpec(2, 12, 12, [cbi.LayerDesc(cbi.LayerKind.Conv, "stem", [], stem, True)])
        for nm in ("left", "right"):
            s = conv_spec(rng, stem.out_channels, cout=4, k=3, stride=1, pad=1)
            spec.layers.append(cbi.LayerDesc(cbi.LayerKind.Conv, nm, ["stem"], s))
        spec.layers.append(cbi.LayerDesc(join, "join", ["left", "right"]))
        spec.layers.append(cbi.LayerDesc(cbi.LayerKind.Conv, "head", [],
                                         conv_spec(rng, 4 if join == cbi.LayerKind.Add else 8, k=3, stride=1,
                                                   pad=1)))
        r, q = oracle.RefNet(spec, [0.0] * 4), oracle.PortNet(spec, [0.0] * 4)
        for t in range(4):
            x = rng.uniform(0, 1, (2, 12, 12)).astype(np.float32)
            assert np.array_equal(r.forward(x), q.forward(x))


# ---------------------------------------------------------------------------
# known-answer vectors from the reference's own tests
# ---------------------------------------------------------------------------
def load_kats():
    with open(os.path.join(HERE, "golden", "kats.json")) as fh:
        return json.load(fh)


@need_port
def test_port_reproduces_reference_kats():
    P = oracle.port()
    k = load_kats()
    for case in k["detect"]:
        x = np.array(case["x"], np.float32).reshape(case["shape"])
        st = np.array(case["state"], np.float32).reshape(case["shape"])
        m = np.zeros(case["shape"][1:], np.uint8)
        P.cbo_detect_changes(p(x), p(st), *case["shape"], case["tau"], case["mode"], p(m))
        assert m.ravel().tolist() == case["map"], case["ref"]
        assert np.allclose(st.ravel(), case["state_after"]), case["ref"]
    for case in k["dilate"]:
        h, w = case["in"]
        m = np.zeros((h, w), np.uint8)
        for (j, i) in case["set"]:
            m[j, i] = 1
        oh, ow = case["out"]
        d = np.zeros((oh, ow), np.uint8)
        P.cbo_dilate_window(p(m), h, w, case["k"], case["k"], case["stride"], case["pad"], oh, ow, p(d))
        assert int(d.sum()) == case["count"], case["ref"]
        for (j, i) in case.get("marked", []):
            assert d[j, i] == 1, case["ref"]
    for case in k["conv"]:
        spec = cbi.ConvSpec(1, 1, 3, 3, 1, case["pad"])
        spec.weights = np.ones(9, np.float32)
        spec.bias = np.zeros(1, np.float32)
        keep = []
        cs = spec._c(keep)
        x = np.arange(1, 10, dtype=np.float32).reshape(1, 3, 3)
        y = np.zeros((1, 3, 3), np.float32)
        P.cbo_conv2d_dense(p(x), 1, 3, 3, C.byref(cs), p(y))
        for (j, i, v) in case["values"]:
            assert y[0, j, i] == v, case["ref"]
        col = np.zeros(9, np.float32)
        P.cbo_im2col(p(x), 1, 3, 3, C.byref(cs), p(np.array([[0, 0]], np.int32)), 1, p(col))
        assert col.tolist() == case["im2col_00"], case["ref"]
    for case in k["pool"]:
        x = np.array(case["x"], np.float32).reshape(case["shape"])
        c, h, w = case["shape"]
        oh, ow = case["out"]
        y = np.zeros((c, oh, ow), np.float32)
        P.cbo_maxpool_to(p(x), c, h, w, 2, 2, oh, ow, p(y))
        assert y.ravel().tolist() == case["y"], case["ref"]
    g = k["gemm"]
    spec = cbi.ConvSpec(2, 2, 1, 1, 1, 0)
    spec.weights = np.array(g["K"], np.float32)
    spec.bias = np.zeros(2, np.float32)
    keep = []
    cs = spec._c(keep)
    y = np.zeros(2, np.float32)
    P.cbo_gemm(C.byref(cs), p(np.array(g["x"], np.float32)), 1, p(y))
    assert y.tolist() == g["y"], g["ref"]


# ---------------------------------------------------------------------------
# product harness == reference harness (inputs are identical on both sides)
# ---------------------------------------------------------------------------
@need_ref
@pytest.mark.parametrize("cfg", [
    cbi.SyntheticConfig(32, 40, 3, 5, 2, 6, 2, 3, 0.0, 7),
    cbi.SyntheticConfig(48, 48, 2, 4, 3, 9, 4, 1, 0.01, 21),
    cbi.SyntheticConfig(20, 64, 1, 6, 1, 20, 5, 5, 0.08, 701),
])
def test_gen_synthetic_matches_reference(cfg):
    a, ca = cbi.gen_synthetic(cfg, with_corners=True)
    b, cb = oracle.ref_gen_synthetic(cfg, with_corners=True)
    assert np.array_equal(a, b) and np.array_equal(ca, cb)


@need_ref
def test_fill_random_weights_matches_reference():
    spec = cbi.make_seg_spec(1, 64, 64)
    want = oracle.ref_fill_random_weights(cbi.make_seg_spec(1, 64, 64), 1)
    got = [(d.conv.weights, d.conv.bias) for d in spec.layers if d.kind == cbi.LayerKind.Conv]
    for (gw, gb), (ww, wb) in zip(got, want):
        assert np.array_equal(gw, ww) and np.array_equal(gb, wb)


def test_golden_sequence_fixture_matches_port():
    """tests/golden/seq_small.npz: frames + reference outputs generated by
    tests/golden/make_golden.py from the reference build; the port must
    reproduce the recorded outputs and layer-1 index lists bit-for-bit."""
    path = os.path.join(HERE, "golden", "seq_small.npz")
    if not os.path.exists(path) or not oracle.port_available():
        pytest.skip("golden fixture or port not available")
    z = np.load(path)
    spec = cbi.make_seg_spec(int(z["seed"]), int(z["height"]), int(z["width"]))
    q = oracle.PortNet(spec, list(z["taus"]))
    for t in range(z["frames"].shape[0]):
        assert np.array_equal(q.forward(z["frames"][t]), z["outputs"][t])
        _, idx = q.changes(0)
        n = int(z["l1_count"][t])
        assert np.array_equal(idx, z["l1_idx"][t, :n])


# ---------------------------------------------------------------------------
# EXTENSIONS beyond the reference (leaky ReLU, upsampling): parity unpinned
# against the reference, so the C restatement is checked against an
# independent float64 numpy formulation instead (tests/oracle.py dense_forward64)
# ---------------------------------------------------------------------------
def test_reference_rejects_the_extensions():
    spec = cbi.make_yolov3_spec(3, 64, 96, width_div=16)
    with pytest.raises(cbi.ConfigError):
        oracle.RefNet(spec, [0.0] * 13)


@pytest.mark.parametrize("seed", [1, 2])
def test_extensions_port_matches_float64_dense(seed):
    """YOLOv3-style graph (leaky convs, ceil pools, x2 upsample + concat route)
    at tau = 0: every frame the CB restatement equals the float64 dense net
    (acceptance C1's property), and its change maps cover every pixel whose
    dense output moved."""
    rng = np.random.default_rng(seed)
    spec = cbi.make_yolov3_spec(seed, 72, 104, width_div=16)
    net = oracle.PortNet(spec, [0.0] * 13)
    rows = {d.name: i for i, d in enumerate(spec.layers)}
    x = rng.uniform(0, 1, (3, 72, 104)).astype(np.float32)
    prev = None
    for t in range(4):
        net.forward(x)
        dense = oracle.dense_forward64(spec, x)
        for node, name in enumerate(n for n in (d.name for d in spec.layers)):
            want = dense[rows[name]]
            got = net.output(node)
            assert got.shape == want.shape, name
            err = np.abs(got - want).max() / max(1e-30, np.abs(want).max())
            assert err < 2e-5, (t, name, err)
        if prev is not None:  # changed output pixels are marked (tau = 0: exactly the moved ones or more)
            node = [d.name for d in spec.layers].index("up")
            m, _ = net.changes(node)
            moved = np.any(dense[rows["up"]] != prev[rows["up"]], axis=0)
            assert not np.any(moved & (m == 0))
        prev = dense
        x = x.copy()
        j, i = rng.integers(0, 60), rng.integers(0, 90)
        x[:, j:j + 9, i:i + 11] = rng.uniform(0, 1, (3, 9, 11)).astype(np.float32)


def test_leaky_slope_on_a_single_conv():
    """fused leaky ReLU: v < 0 ? v * slope : v with one fp32 rounding (Darknet's leaky)"""
    rng = np.random.default_rng(5)
    cs = cbi.ConvSpec(4, 6, 3, 3, 1, 1, 0, 0, rng.normal(0, 1, 6 * 4 * 9).astype(np.float32),
                      rng.normal(0, 1, 6).astype(np.float32))
    spec = cbi.NetworkSpec(4, 10, 12, [cbi.LayerDesc(cbi.LayerKind.Conv, "c", [], cs, False),
                                       cbi.LayerDesc(cbi.LayerKind.Act, "a", act_slope=0.1)])
    lin = cbi.NetworkSpec(4, 10, 12, [cbi.LayerDesc(cbi.LayerKind.Conv, "c", [], cs, False)])
    x = rng.uniform(-1, 1, (4, 10, 12)).astype(np.float32)
    a, b = oracle.PortNet(spec, [0.0]), oracle.PortNet(lin, [0.0])
    ya, yb = a.forward(x), b.forward(x)
    want = np.where(yb < 0, yb * np.float32(0.1), yb).astype(np.float32)
    assert np.array_equal(ya, want)
    assert np.any(yb < 0)
