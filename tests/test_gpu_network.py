"""GPU parity: CBNetwork (multi-stream, CUDA-graph frame step) vs the reference
CBNetwork on identical gen_synthetic sequences.

Parity contract: layer-1 change maps / index lists bit-exact
frame by frame; per-layer mask agreement reported for deeper layers; final
maps within max_rel_err <= TOL_NET.
"""
import numpy as np
import pytest

from paper_1808_05488_b200 import _lib, cbi
from tests import oracle

pytestmark = pytest.mark.gpu

TOL_NET = 8e-5  # 2x the largest observed (4.0e-5, test_pnm8_state_shadow_mixed_ingest; CBG_PARITY_OUT)


def seq(h, w, n=6, seed=7, objects=3, size=10, vel=3, noise=0.0, c=3):
    return cbi.gen_synthetic(cbi.SyntheticConfig(h, w, c, n, objects, size, vel, vel, noise, seed))


def compare_run(spec, taus, frames, policies=None, mode=cbi.DetectMode.ClosedLoop, tol=TOL_NET):
    net = cbi.convert_to_cb(spec, taus, policies, mode)
    ref = oracle.RefNet(spec, taus, policies, mode)
    agree = []
    for t, f in enumerate(frames):
        got = net.forward_frame(f)
        want = ref.forward(f)
        for i in range(len(net.nodes())):
            gm, gi = net.node_changes(i)
            st = ref.stats(i)
            if i == 0:
                assert np.array_equal(gm, st["map"]), f"frame {t}: layer-1 map differs"
                assert len(gi) == st["changed_px"]
            agree.append(float(np.mean(gm == st["map"])))
        err = oracle.max_rel_err(got, want)
        assert err <= tol, f"frame {t}: max_rel_err {err}"
    return net, ref, agree


def test_seg_net_small_resolution(gpu):
    spec = cbi.make_seg_spec(1, 96, 128)
    net, ref, agree = compare_run(spec, [0.05] * 5, seq(96, 128))
    assert min(agree) >= 0.999


def test_seg_net_every_node_matches(gpu):
    spec = cbi.make_seg_spec(3, 80, 96)
    taus = [0.04, 0.05, 0.05, 0.03, 0.02]
    net = cbi.convert_to_cb(spec, taus)
    ref = oracle.RefNet(spec, taus)
    for t, f in enumerate(seq(80, 96, n=5, seed=11, noise=0.004)):
        net.forward_frame(f)
        ref.forward(f)
        for i, n in enumerate(net.nodes()):
            assert oracle.max_rel_err(net.node_output(i), ref.output(i)) <= TOL_NET, (t, n.name)
        gm, gi = net.node_changes(0)
        wm = ref.stats(0)["map"]
        assert np.array_equal(gm, wm)
        assert np.array_equal(gi, np.argwhere(wm).astype(np.int32))


def test_zero_threshold_equivalence_to_dense(gpu):
    """acceptance C1: tau = 0 => CB output == dense output (within TOL)."""
    rng = np.random.default_rng(101)
    for rnd in range(6):
        h, w = int(rng.integers(12, 33)), int(rng.integers(12, 33))
        spec = cbi.make_small_spec(int(rng.integers(1, 1000)), 2, h, w)
        net = cbi.convert_to_cb(spec, [0.0] * 3)
        ref = oracle.RefNet(spec, [0.0] * 3)
        x = rng.uniform(0, 1, (2, h, w)).astype(np.float32)
        for t in range(6):
            got = net.forward_frame(x)
            assert oracle.max_rel_err(got, ref.dense_forward(x)) <= 2e-5
            x = x.copy()
            n = int(rng.integers(0, h * w // 8 + 1))
            x[:, rng.integers(0, h, n), rng.integers(0, w, n)] = rng.uniform(0, 1, (2, n)).astype(np.float32)


def test_multi_stream_matches_independent_references(gpu):
    """S streams in one stream set == S independent reference CBNetworks."""
    S, H, W = 3, 64, 80
    spec = cbi.make_seg_spec(5, H, W)
    taus = [0.05] * 5
    seqs = [seq(H, W, n=4, seed=1000 + s) for s in range(S)]
    net = cbi.convert_to_cb(spec, taus, n_streams=S)
    refs = [oracle.RefNet(spec, taus) for _ in range(S)]
    for t in range(4):
        batch = np.stack([seqs[s][t] for s in range(S)])
        net.enqueue(batch)
        counts = net.counts()
        for s in range(S):
            want = refs[s].forward(seqs[s][t])
            assert oracle.max_rel_err(net.output(s), want) <= TOL_NET
            assert counts[0, s] == refs[s].stats(0)["changed_px"]


def test_reset_and_thresholds(gpu):
    spec = cbi.make_small_spec(6, 2, 32, 32)
    frames = seq(32, 32, n=6, seed=9, objects=1, size=6, vel=1, noise=0.01, c=2)
    net = cbi.convert_to_cb(spec, [0.02] * 3)
    a = [net.forward_frame(f).copy() for f in frames]
    ca = [net.counts().copy() for _ in range(1)]
    net.reset()
    b = [net.forward_frame(f).copy() for f in frames]
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    # thresholds: lower tau without reset must re-detect exactly like the reference
    ref = oracle.RefNet(spec, [0.02] * 3)
    net2 = cbi.convert_to_cb(spec, [0.02] * 3)
    for f in frames[:3]:
        ref.forward(f)
        net2.forward_frame(f)
    ref.set_thresholds([0.001, 0.001, 0.001])
    net2.set_thresholds([0.001, 0.001, 0.001])
    assert net2.thresholds() == pytest.approx([0.001] * 3)
    for f in frames[3:]:
        want = ref.forward(f)
        got = net2.forward_frame(f)
        for i in range(len(net2.nodes())):
            assert len(net2.node_changes(i)[1]) == ref.stats(i)["changed_px"]
        assert oracle.max_rel_err(got, want) <= TOL_NET
    del ca


def test_identical_second_frame_changes_nothing(gpu):
    """test_network.cpp:108-128 at pinned seg7 dims (776x1040)."""
    spec = cbi.make_seg7_spec(3)
    net = cbi.convert_to_cb(spec, [0.0] * 5)
    rng = np.random.default_rng(41)
    frame = rng.uniform(0, 1, (3, 776, 1040)).astype(np.float32)
    out = net.forward_frame(frame)
    assert out.shape == (8, 136, 218) and np.all(np.isfinite(out))
    net.forward_frame(frame)
    assert np.all(net.counts() == 0)


def test_narrow_layers_bit_exact(gpu):
    """Layers with Cout <= 16 run the CUDA-core path (conv_exact.cu) in the
    reference's own summation order: the first layer's retained output, the
    pool after it and the next layer's change maps are bit-identical to the
    reference, frame by frame (SURVEY.md §8c asks for <= 1e-5 there)."""
    H, W = 96, 128
    spec = cbi.make_seg_spec(2, H, W)
    taus = [0.05] * 5
    net = cbi.convert_to_cb(spec, taus)
    ref = oracle.RefNet(spec, taus)
    for t, f in enumerate(seq(H, W, n=6, seed=21, noise=0.002)):
        net.forward_frame(f)
        ref.forward(f)
        assert np.array_equal(net.node_output(0), ref.output(0)), f"frame {t}: L1 output not bit-exact"
        assert np.array_equal(net.node_output(1), ref.output(1)), f"frame {t}: L2b output not bit-exact"
        gm, _ = net.node_changes(2)
        assert np.array_equal(gm, ref.stats(2)["map"]), f"frame {t}: L3 map differs"
        assert np.array_equal(net.node_state(2), ref.state(2, net.nodes()[2].in_shape)), f"frame {t}: L3 state differs"


def test_pnm8_ingest_matches_fp32_and_reference(gpu):
    """8-bit frames in PNM payload order (cbg_net_forward_u8) are converted on
    the device exactly as load_pnm does (byte / 255.0f): the run is bit-identical
    to the fp32 API fed with from_pnm8(frames), and matches the reference on them."""
    S, H, W = 2, 64, 80
    spec = cbi.make_seg_spec(4, H, W)
    taus = [0.05] * 5
    raw = np.stack([seq(H, W, n=5, seed=300 + s, noise=0.01) for s in range(S)], axis=1)
    pnm = cbi.to_pnm8(raw)                      # [T, S, H, W, C] uint8
    f32 = cbi.from_pnm8(pnm)                    # [T, S, C, H, W] = byte / 255
    assert np.array_equal(f32[..., :4, :4], (pnm.astype(np.float32) / np.float32(255)).transpose(0, 1, 4, 2, 3)[..., :4, :4])
    a = cbi.convert_to_cb(spec, taus, n_streams=S)
    b = cbi.convert_to_cb(spec, taus, n_streams=S)
    refs = [oracle.RefNet(spec, taus) for _ in range(S)]
    for t in range(len(pnm)):
        a.enqueue_u8(pnm[t])
        b.enqueue(f32[t])
        assert np.array_equal(a.counts(), b.counts())
        for s in range(S):
            assert np.array_equal(a.output(s), b.output(s))
            assert np.array_equal(a.node_state(0, s), b.node_state(0, s))
            want = refs[s].forward(f32[t, s])
            assert np.array_equal(a.node_output(0, s), refs[s].output(0))  # first layer bit-exact
            assert oracle.max_rel_err(a.output(s), want) <= TOL_NET


def test_pnm8_state_shadow_mixed_ingest(gpu):
    """The 8-bit ingest keeps a byte shadow of the first layer's state and
    compares against it once every stream had a full update through the 8-bit
    path. Mixed feeding (8-bit, fp32, 8-bit again, a per-stream reset, a forced
    full update) must stay bit-identical to the fp32 API on the same values and
    to the reference, whichever comparison source each frame used."""
    S, H, W = 3, 48, 64
    spec = cbi.make_seg_spec(5, H, W)
    taus = [0.04] * 5
    raw = np.stack([seq(H, W, n=12, seed=700 + s, noise=0.02) for s in range(S)], axis=1)
    pnm = cbi.to_pnm8(raw)
    f32 = cbi.from_pnm8(pnm)
    a = cbi.convert_to_cb(spec, taus, n_streams=S)
    b = cbi.convert_to_cb(spec, taus, n_streams=S)
    refs = [oracle.RefNet(spec, taus) for _ in range(S)]
    # frame -> how net a is fed: u8, f32, u8 + reset of stream 1 before, u8 + FORCE_FULL
    plan = ["u8", "u8", "u8", "f32", "u8", "u8", "reset1", "u8", "u8", "full", "u8", "u8"]
    for t, how in enumerate(plan):
        if how == "reset1":
            a.reset(1)
            b.reset(1)
            refs[1].reset()
        if how == "f32":
            a.enqueue(f32[t])
        elif how == "full":
            a.enqueue_u8(pnm[t], _lib.FWD_FORCE_FULL)
        else:
            a.enqueue_u8(pnm[t])
        b.enqueue(f32[t], _lib.FWD_FORCE_FULL if how == "full" else 0)
        assert np.array_equal(a.counts(), b.counts()), (t, how)
        for s in range(S):
            if how == "full":
                refs[s].reset()
            want = refs[s].forward(f32[t, s])
            assert np.array_equal(a.node_state(0, s), b.node_state(0, s)), (t, s)
            assert np.array_equal(a.node_output(0, s), refs[s].output(0)), (t, s)
            assert np.array_equal(a.output(s), b.output(s)), (t, s)
            assert oracle.max_rel_err(a.output(s), want) <= TOL_NET


def test_bench_workload_parity(gpu):
    """The bench's own workload at full size (seg net 640x480, tau 0.05, PNM-
    quantized gen_synthetic seeds 1000/1001, 6 objects of 40 px, v = 4), two
    streams in one set through the 8-bit ingest, against the reference on the
    same frames: layers 1-3 bit-exact (maps, lists, L1/L2b outputs), final maps
    within TOL, every deeper map >= 99.9% equal (measured: all equal except one
    L5 pixel of 18.6k on one frame, a tau crossing inside the fp32-accurate
    3xFP16 rounding)."""
    H, W, S, T = 480, 640, 2, 4
    spec = cbi.make_seg_spec(1, H, W)
    taus = [0.05] * 5
    pnm = np.stack([cbi.to_pnm8(cbi.gen_synthetic(cbi.SyntheticConfig(H, W, 3, T, 6, 40, 4, 4, 0.0, 1000 + s)))
                    for s in range(S)], axis=1)
    f32 = cbi.from_pnm8(pnm)
    net = cbi.convert_to_cb(spec, taus, n_streams=S)
    refs = [oracle.RefNet(spec, taus) for _ in range(S)]
    for t in range(T):
        net.enqueue_u8(pnm[t])
        counts = net.counts()
        for s in range(S):
            want = refs[s].forward(f32[t, s])
            assert oracle.max_rel_err(net.output(s), want) <= TOL_NET, (t, s)
            assert np.array_equal(net.node_output(0, s), refs[s].output(0)), (t, s)
            assert np.array_equal(net.node_output(1, s), refs[s].output(1)), (t, s)
            for i in range(len(net.nodes())):
                gm, _ = net.node_changes(i, s)
                wm = refs[s].stats(i)["map"]
                if i <= 2:
                    assert np.array_equal(gm, wm) and counts[i, s] == refs[s].stats(i)["changed_px"], (t, s, i)
                else:
                    assert float(np.mean(gm == wm)) >= 0.999, (t, s, i)


def test_presplit_copy_follows_growing_magnitudes(gpu, monkeypatch):
    """The detect of a 3xFP16 k x k layer keeps its state pre-split with the
    GEMM's exponent; when the operand bound grows (frames brighten in 4x
    steps, so every layer's running |max| and exponent move) the detect
    rewrites the whole copy that frame. The network must be bit-identical to
    one built with CBG_PRESPLIT=0 (the GEMM splitting the fp32 state itself,
    same exponent, same arithmetic) on every node, and layers 1-3 must match
    the reference's counts."""
    S, H, W = 2, 56, 72
    spec = cbi.make_seg_spec(8, H, W)
    taus = [0.02] * 5
    base = np.stack([seq(H, W, n=7, seed=900 + s, noise=0.01) for s in range(S)], axis=1)
    gain = np.float32([1, 1, 4, 4, 16, 16, 64]).reshape(-1, 1, 1, 1, 1)
    frames = (base * gain).astype(np.float32)
    net = cbi.convert_to_cb(spec, taus, n_streams=S)
    monkeypatch.setenv("CBG_PRESPLIT", "0")
    plain = cbi.convert_to_cb(spec, taus, n_streams=S)
    refs = [oracle.RefNet(spec, taus) for _ in range(S)]
    for t in range(len(frames)):
        net.enqueue(frames[t])
        plain.enqueue(frames[t])
        counts = net.counts()
        assert np.array_equal(counts, plain.counts()), t
        for s in range(S):
            refs[s].forward(frames[t, s])
            for i in range(len(net.nodes())):
                assert np.array_equal(net.node_output(i, s), plain.node_output(i, s)), (t, s, i)
            for i in range(3):
                assert counts[i, s] == refs[s].stats(i)["changed_px"], (t, s, i)


def test_presplit_copy_under_control_operations(gpu, monkeypatch):
    """Pre-split vs GEMM-side split, bit-identical on every node while the
    sequence goes through the control paths that change which pixels the
    detect walks: a threshold decrease (dense rescan), a per-stream reset, a
    forced full update, dense mode on and off, and 8-bit frames."""
    S, H, W, T = 3, 48, 64, 12
    spec = cbi.make_seg_spec(9, H, W)
    taus = [0.05] * 5
    raw = np.stack([seq(H, W, n=T, seed=950 + s, noise=0.02) for s in range(S)], axis=1)
    pnm = cbi.to_pnm8(raw)
    f32 = cbi.from_pnm8(pnm)
    net = cbi.convert_to_cb(spec, taus, n_streams=S)
    monkeypatch.setenv("CBG_PRESPLIT", "0")
    plain = cbi.convert_to_cb(spec, taus, n_streams=S)
    for t in range(T):
        for n_ in (net, plain):
            if t == 3:
                n_.set_thresholds([0.02] * 5)   # tau decreased: dense rescan next frame
            if t == 5:
                n_.reset(2)
            if t == 7:
                n_.set_dense(True)
            if t == 9:
                n_.set_dense(False)
            if t % 2:
                n_.enqueue_u8(pnm[t])
            else:
                n_.enqueue(f32[t], _lib.FWD_FORCE_FULL if t == 6 else 0)
        assert np.array_equal(net.counts(), plain.counts()), t
        for s in range(S):
            for i in range(len(net.nodes())):
                assert np.array_equal(net.node_output(i, s), plain.node_output(i, s)), (t, s, i)
