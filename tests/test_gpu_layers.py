"""GPU parity: standalone CBConvLayer / CBPoolLayer through the C ABI vs the
reference build (oracle/_ref), on identical seeded inputs.

Adapted from the reference's tests/test_layers.cpp and acceptance C1-C3.
Bars: change maps, index lists, input states and pooled
outputs are bit-exact; conv outputs (3xFP16 tcgen05 GEMM with a different sum
order than the reference's sequential fp32 loop, or bit-exact on the CUDA-core
path for Cout <= 16) within max_rel_err (tests/oracles.hpp:59-66) <= TOL.
"""
import numpy as np
import pytest

from paper_1808_05488_b200 import cbi
from tests import oracle

pytestmark = pytest.mark.gpu

TOL = 4e-6  # max_rel_err for conv outputs: 2x the largest observed (1.97e-6; CBG_PARITY_OUT)


def rand_spec(rng, cin, kernels=(1, 3, 5, 7), max_out=40, stride=None, pad=None):
    k = int(rng.choice(kernels))
    s = cbi.ConvSpec(cin, int(rng.integers(1, max_out + 1)), k, k,
                     int(stride if stride is not None else rng.integers(1, 3)),
                     int(pad if pad is not None else rng.integers(0, k // 2 + 1)))
    a = 1.0 / np.sqrt(cin * k * k)
    s.weights = rng.uniform(-a, a, s.weight_count()).astype(np.float32)
    s.bias = rng.uniform(-0.1, 0.1, s.out_channels).astype(np.float32)
    return s


def pair(spec, tau, policy=cbi.DetectionPolicy.Detect, relu=False, mode=cbi.DetectMode.ClosedLoop, h=16, w=16):
    g = cbi.CBConvLayer(spec, tau, policy, relu, mode, h, w)
    r = oracle.RefConv(spec, tau, policy, relu, mode, h, w)
    return g, r


def same_changes(res, r):
    m, idx = r.changes()
    assert np.array_equal(res.out_map, m)
    assert np.array_equal(res.indexes, idx)


def test_cfg1_single_cbconv_block_change(gpu):
    """BASELINE configs[0]: CBconv 3x3 16->32, 64x64, ~5% changed output pixels."""
    rng = np.random.default_rng(1)
    spec = rand_spec(rng, 16, kernels=(3,), stride=1, pad=1)
    spec.out_channels = 32
    spec.weights = rng.uniform(-0.08, 0.08, spec.weight_count()).astype(np.float32)
    spec.bias = rng.uniform(-0.05, 0.05, 32).astype(np.float32)
    g, r = pair(spec, 0.05, h=64, w=64)
    a = cbi.gen_synthetic(cbi.SyntheticConfig(64, 64, 16, 1, 0, 8, seed=7))[0]
    b = a.copy()
    b[:, 20:32, 30:42] = rng.uniform(0, 1, (16, 12, 12)).astype(np.float32)
    for x, force in ((a, True), (b, False), (a, False), (b, False)):
        res = g.forward(x, force_full_update=force)
        eff = r.forward(x, force=force)
        same_changes(res, r)
        assert res.eff_ops == eff
        assert np.array_equal(g.state, r.state)
        assert oracle.max_rel_err(g.prev_output, r.prev_output) <= TOL
    assert len(res.indexes) == 14 * 14  # 12x12 block dilated by the 3x3 support


@pytest.mark.parametrize("seed", range(12))
def test_random_detect_layers_match_reference(gpu, seed):
    rng = np.random.default_rng(100 + seed)
    cin = int(rng.integers(1, 9))
    h, w = int(rng.integers(7, 30)), int(rng.integers(7, 30))
    spec = rand_spec(rng, cin)
    try:
        spec.output_height(h), spec.output_width(w)
    except cbi.InvalidInputError:
        return
    if rng.random() < 0.3:  # pinned dims behave as a crop (tensor.hpp:49-53)
        spec.out_h = max(1, spec.output_height(h) - int(rng.integers(0, 3)))
        spec.out_w = max(1, spec.output_width(w) - int(rng.integers(0, 3)))
    tau = float(rng.choice([0.0, 0.02, 0.1]))
    relu = bool(rng.integers(0, 2))
    mode = cbi.DetectMode(int(rng.integers(0, 2)))
    g, r = pair(spec, tau, relu=relu, mode=mode, h=h, w=w)
    x = rng.uniform(0, 1, (cin, h, w)).astype(np.float32)
    for t in range(5):
        res = g.forward(x, force_full_update=(t == 0))
        eff = r.forward(x, force=(t == 0))
        same_changes(res, r)
        assert res.eff_ops == eff
        assert np.array_equal(g.state, r.state)
        assert oracle.max_rel_err(g.prev_output, r.prev_output) <= TOL
        x = x.copy()
        n = int(rng.integers(0, h * w // 4 + 1))
        jj, ii = rng.integers(0, h, n), rng.integers(0, w, n)
        x[:, jj, ii] += rng.uniform(-0.2, 0.2, (cin, n)).astype(np.float32)


def test_bootstrap_full_update_equals_dense(gpu):
    """test_layers.cpp:76-89: bootstrap == conv2d_dense."""
    rng = np.random.default_rng(23)
    for _ in range(5):
        spec = rand_spec(rng, 2, stride=1)
        relu = bool(rng.integers(0, 2))
        g, r = pair(spec, 0.0, relu=relu, h=9, w=9)
        x = rng.uniform(-1, 1, (2, 9, 9)).astype(np.float32)
        res = g.forward(x, force_full_update=True)
        r.forward(x, force=True)
        assert len(res.indexes) == g.out_h * g.out_w
        assert oracle.max_rel_err(g.prev_output, r.prev_output) <= TOL


def test_repeated_frame_costs_zero_ops(gpu):
    """test_layers.cpp:63-74."""
    rng = np.random.default_rng(22)
    spec = rand_spec(rng, 3, stride=1)
    g, _ = pair(spec, 0.0, h=10, w=10)
    x = rng.uniform(-1, 1, (3, 10, 10)).astype(np.float32)
    g.forward(x, force_full_update=True)
    before = g.prev_output
    res = g.forward(x)
    assert len(res.indexes) == 0 and res.eff_ops == 0
    assert np.array_equal(g.prev_output, before)


def test_single_pixel_change_updates_kernel_support(gpu):
    """test_layers.cpp:91-107: 7x7 kernel, one interior pixel -> exactly 49 outputs."""
    rng = np.random.default_rng(24)
    spec = rand_spec(rng, 1, kernels=(7,), stride=1, pad=3)
    g, _ = pair(spec, 0.0, h=12, w=12)
    x = rng.uniform(-1, 1, (1, 12, 12)).astype(np.float32)
    g.forward(x, force_full_update=True)
    x[0, 6, 6] += 1.0
    assert len(g.forward(x).indexes) == 49


def test_closed_loop_consistency(gpu):
    """test_layers.cpp:109-121 / acceptance C2: prev_output == conv(state)."""
    rng = np.random.default_rng(25)
    spec = rand_spec(rng, 2, stride=1)
    g, r = pair(spec, 0.05, h=8, w=8)
    x = rng.uniform(-1, 1, (2, 8, 8)).astype(np.float32)
    g.forward(x, force_full_update=True)
    r.forward(x, force=True)
    for _ in range(6):
        x = (x + rng.uniform(-0.1, 0.1, x.shape)).astype(np.float32)
        g.forward(x)
        r.forward(x)
        assert np.array_equal(g.state, r.state)
        full = cbi.CBConvLayer(spec, 0.0, in_height=8, in_width=8)
        full.forward(g.state, force_full_update=True)
        assert oracle.max_rel_err(g.prev_output, full.prev_output) <= TOL


def test_propagate_and_reuse_policies(gpu):
    rng = np.random.default_rng(29)
    s1 = rand_spec(rng, 2, kernels=(3,), stride=1, pad=1)
    s2 = rand_spec(rng, s1.out_channels, kernels=(3,), stride=1, pad=1)
    a = cbi.CBConvLayer(s1, 0.0, in_height=8, in_width=8)
    b = cbi.CBConvLayer(s2, 0.0, cbi.DetectionPolicy.Propagate, in_height=8, in_width=8)
    rb = oracle.RefConv(s2, 0.0, cbi.DetectionPolicy.Propagate, in_h=8, in_w=8)
    x = rng.uniform(-1, 1, (2, 8, 8)).astype(np.float32)
    ra = a.forward(x, force_full_update=True)
    b.forward(a.prev_output, cbi.UpstreamChange(ra.out_map, ra.indexes), force_full_update=True)
    rb.forward(a.prev_output, ra.out_map, ra.indexes, force=True)
    for _ in range(4):
        x[int(rng.integers(0, 2)), int(rng.integers(0, 8)), int(rng.integers(0, 8))] += 0.5
        ra = a.forward(x)
        up = cbi.UpstreamChange(ra.out_map, ra.indexes)
        res = b.forward(a.prev_output, up, record_worst_case=True)
        rb.forward(a.prev_output, ra.out_map, ra.indexes, worst=True)
        same_changes(res, rb)
        wm, wn = rb.worst_case()
        assert np.array_equal(res.worst_case_map, wm) and res.propagated_px == wn
        assert oracle.max_rel_err(b.prev_output, rb.prev_output) <= TOL
    # reuse_1x1: upstream map and indexes used verbatim (layers.cpp:96-104)
    s3 = cbi.ConvSpec(s1.out_channels, 5, 1, 1, 1, 0)
    s3.weights = rng.uniform(-0.5, 0.5, s3.weight_count()).astype(np.float32)
    s3.bias = rng.uniform(-0.1, 0.1, 5).astype(np.float32)
    c = cbi.CBConvLayer(s3, 0.0, cbi.DetectionPolicy.Reuse1x1, True, in_height=8, in_width=8)
    rc = oracle.RefConv(s3, 0.0, cbi.DetectionPolicy.Reuse1x1, True, in_h=8, in_w=8)
    c.forward(a.prev_output, force_full_update=True)
    rc.forward(a.prev_output, force=True)
    x[0, 3, 3] -= 0.7
    ra = a.forward(x)
    res = c.forward(a.prev_output, cbi.UpstreamChange(ra.out_map, ra.indexes))
    rc.forward(a.prev_output, ra.out_map, ra.indexes)
    same_changes(res, rc)
    assert oracle.max_rel_err(c.prev_output, rc.prev_output) <= TOL


def test_policy_errors(gpu):
    rng = np.random.default_rng(27)
    prop = cbi.CBConvLayer(rand_spec(rng, 2, stride=1), 0.0, cbi.DetectionPolicy.Propagate, in_height=8,
                           in_width=8)
    with pytest.raises(cbi.ConfigError):
        prop.forward(np.zeros((2, 8, 8), np.float32))
    s = rand_spec(rng, 2, kernels=(3,), pad=1)
    with pytest.raises(cbi.ConfigError):
        cbi.CBConvLayer(s, 0.0, cbi.DetectionPolicy.Reuse1x1, in_height=8, in_width=8)
    with pytest.raises(cbi.InvalidInputError):
        cbi.CBConvLayer(s, -0.1, in_height=8, in_width=8)


def test_pool_layers_bit_exact(gpu):
    """test_layers.cpp:189-227: CB pool == reference pool, including ceil-mode dims."""
    rng = np.random.default_rng(31)
    x = rng.uniform(-1, 1, (3, 9, 7)).astype(np.float32)
    for (oh, ow) in ((4, 3), (5, 4)):  # floor-mode and ceil-mode (clipped windows)
        g = cbi.CBPoolLayer(2, 2, 3, 9, 7, oh, ow)
        r = oracle.RefPool(2, 2, 3, 9, 7, oh, ow)
        g.forward(x, force_full_update=True)
        r.forward(x, force=True)
        assert np.array_equal(g.prev_output, r.prev_output)
        for _ in range(4):
            m = (rng.random((9, 7)) < 0.1).astype(np.uint8)
            x = np.where(m[None], rng.uniform(-1, 1, x.shape), x).astype(np.float32)
            idx = np.argwhere(m).astype(np.int32)
            res = g.forward(x, cbi.UpstreamChange(m, idx))
            r.forward(x, m, idx)
            rm, ri = r.changes()
            assert np.array_equal(res.out_map, rm) and np.array_equal(res.indexes, ri)
            assert np.array_equal(g.prev_output, r.prev_output)
    with pytest.raises(cbi.ConfigError):
        cbi.CBPoolLayer(2, 2, 1, 4, 4, 2, 2).forward(np.zeros((1, 4, 4), np.float32))


@pytest.mark.parametrize("prec", ["f16", "tf32"])
@pytest.mark.parametrize("scale", [1.0, 3.0e4, 2.0e-5])
def test_tensor_precisions_and_operand_scaling(gpu, monkeypatch, prec, scale):
    """Both tcgen05 operand splits (3xFP16 with power-of-two scaling, the
    default, and 3xTF32) are fp32-accurate over magnitudes far outside fp16's
    range: inputs scaled by 3e4 (fp16 would overflow unscaled) and 2e-5 (the
    lo parts would be subnormal unscaled). Error is measured relative to the
    output's magnitude."""
    monkeypatch.setenv("CBG_GEMM_PREC", prec)
    rng = np.random.default_rng(77)
    spec = rand_spec(rng, 24, kernels=(3,), stride=1, pad=1)
    spec.out_channels = 48
    a = 1.0 / np.sqrt(24 * 9)
    spec.weights = rng.uniform(-a, a, spec.weight_count()).astype(np.float32)
    spec.bias = (scale * rng.uniform(-0.1, 0.1, 48)).astype(np.float32)
    g, r = pair(spec, 0.0, h=40, w=36)
    x = (scale * rng.uniform(-1, 1, (24, 40, 36))).astype(np.float32)
    for t in range(3):
        g.forward(x, force_full_update=(t == 0))
        r.forward(x, force=(t == 0))
        want = r.prev_output
        rel = np.max(np.abs(g.prev_output.astype(np.float64) - want)) / np.max(np.abs(want))
        print(f"{prec} scale {scale}: relative error {rel:.3g}")
        assert rel <= 5e-6, f"{prec} scale {scale}: relative error {rel}"
        x = x.copy()
        x[:, rng.integers(0, 40, 50), rng.integers(0, 36, 50)] *= -1.5


def test_epoch_wrap_keeps_upstream_map(gpu):
    """Maps are epoch-tagged and cleared once per 255 frames; the upstream map
    a standalone layer receives on a wrap call must survive the clear. A
    Propagate conv and a pool run 300 calls (past two wraps) against the
    reference, each call changing a few upstream pixels."""
    rng = np.random.default_rng(41)
    s = rand_spec(rng, 3, kernels=(3,), stride=1, pad=1)
    conv = cbi.CBConvLayer(s, 0.0, cbi.DetectionPolicy.Propagate, in_height=12, in_width=10)
    rconv = oracle.RefConv(s, 0.0, cbi.DetectionPolicy.Propagate, in_h=12, in_w=10)
    pool = cbi.CBPoolLayer(2, 2, 3, 12, 10, 6, 5)
    rpool = oracle.RefPool(2, 2, 3, 12, 10, 6, 5)
    x = rng.uniform(-1, 1, (3, 12, 10)).astype(np.float32)
    conv.forward(x, force_full_update=True)
    rconv.forward(x, None, None, force=True)
    pool.forward(x, force_full_update=True)
    rpool.forward(x, force=True)
    for t in range(300):
        m = np.zeros((12, 10), np.uint8)
        m[rng.integers(0, 12, 3), rng.integers(0, 10, 3)] = 1
        x = np.where(m[None], rng.uniform(-1, 1, x.shape), x).astype(np.float32)
        idx = np.argwhere(m).astype(np.int32)
        res = conv.forward(x, cbi.UpstreamChange(m, idx))
        rconv.forward(x, m, idx)
        pres = pool.forward(x, cbi.UpstreamChange(m, idx))
        rpool.forward(x, m, idx)
        if t % 25 == 0 or t in range(250, 260) or t in range(505, 515):
            same_changes(res, rconv)
            rm, ri = rpool.changes()
            assert np.array_equal(pres.out_map, rm) and np.array_equal(pres.indexes, ri), t
            assert np.array_equal(pool.prev_output, rpool.prev_output), t
            assert oracle.max_rel_err(conv.prev_output, rconv.prev_output) <= TOL, t
    assert np.array_equal(pool.prev_output, rpool.prev_output)


@pytest.mark.parametrize("policy", [cbi.DetectionPolicy.Detect, cbi.DetectionPolicy.Propagate])
def test_first_call_without_force_is_not_a_bootstrap(gpu, policy):
    """A standalone layer has no bootstrap (layers.cpp:64-71 runs only under
    force_full_update): the first unforced Detect call compares against the
    zero state, a Propagate call updates only the upstream's dilated pixels."""
    rng = np.random.default_rng(43)
    s = rand_spec(rng, 2, kernels=(3,), stride=1, pad=1)
    g, r = pair(s, 0.05, policy=policy, h=10, w=10)
    x = rng.uniform(0, 1, (2, 10, 10)).astype(np.float32)
    x[:, :5, :] = 0.0  # unchanged against the zero state
    m = np.zeros((10, 10), np.uint8)
    m[7, 3] = 1
    idx = np.argwhere(m).astype(np.int32)
    if policy == cbi.DetectionPolicy.Detect:
        res = g.forward(x)
        r.forward(x)
    else:
        res = g.forward(x, cbi.UpstreamChange(m, idx))
        r.forward(x, m, idx)
    same_changes(res, r)
    assert len(res.indexes) < 100
    assert oracle.max_rel_err(g.prev_output, r.prev_output) <= TOL
    assert np.array_equal(g.prev_output == 0, r.prev_output == 0)
