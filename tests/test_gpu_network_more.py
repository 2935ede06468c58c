"""GPU parity, network level, beyond the basic seg-net runs: detection
policies, feed-forward mode, joins, worst-case propagation, acceptance
criteria C1/C2/C8 (acceptance.cpp:85-123, 402-435), clone, pinned seg7 dims.
Every comparison is against the unmodified reference build on identical inputs.
"""
import ctypes as C

import numpy as np
import pytest

from paper_1808_05488_b200 import _lib, cbi
from tests import oracle
from tests.oracle import p
from tests.test_oracle import conv_spec, random_net

pytestmark = pytest.mark.gpu

TOL = 1e-4  # 2x the largest observed (5.06e-5: the 3xTF32 wide-layer test and the reduced cfg3)


def run_pair(spec, taus, frames, policies=None, mode=cbi.DetectMode.ClosedLoop, worst=False):
    net = cbi.convert_to_cb(spec, taus, policies, mode)
    ref = oracle.RefNet(spec, taus, policies, mode)
    cfg = cbi.StatsConfig(record_worst_case=worst, record_maps=True)
    for t, f in enumerate(frames):
        fs = cbi.FrameStats()
        got = net.forward_frame(f, cfg, fs)
        want = ref.forward(f, record_worst_case=worst)
        assert oracle.max_rel_err(got, want) <= TOL, f"frame {t}"
        for i, row in enumerate(fs.layers):
            st = ref.stats(i)
            if i == 0:
                assert np.array_equal(row.map, st["map"]), f"frame {t}: layer-1 map"
            assert row.changed_px == st["changed_px"], (t, row.layer)
            assert row.eff_ops == st["eff_ops"], (t, row.layer)
            if worst and st["propagated_px"] >= 0:
                assert row.propagated_px == st["propagated_px"], (t, row.layer)
                assert np.array_equal(row.worst_case_map, st["worst_case_map"]), (t, row.layer)
                # C8: the detected set is a subset of the worst-case propagation
                assert not np.any(row.map.astype(bool) & ~row.worst_case_map.astype(bool))
    return net, ref


def frames_for(h, w, n=5, seed=3, c=3, noise=0.0):
    return cbi.gen_synthetic(cbi.SyntheticConfig(h, w, c, n, 3, 10, 3, 3, noise, seed))


def test_policies_propagate_and_reuse(gpu):
    spec = cbi.make_seg_spec(2, 72, 96)
    pol = [cbi.DetectionPolicy.Detect, cbi.DetectionPolicy.Propagate, cbi.DetectionPolicy.Detect,
           cbi.DetectionPolicy.Reuse1x1, cbi.DetectionPolicy.Reuse1x1]
    run_pair(spec, [0.05] * 5, frames_for(72, 96), pol)


def test_feedforward_mode(gpu):
    spec = cbi.make_seg_spec(4, 64, 80)
    run_pair(spec, [0.03] * 5, frames_for(64, 80, noise=0.01), mode=cbi.DetectMode.FeedForward)


def test_worst_case_stats_and_superset(gpu):
    spec = cbi.make_seg_spec(5, 64, 80)
    run_pair(spec, [0.02, 0.05, 0.05, 0.01, 0.01], frames_for(64, 80, noise=0.004), worst=True)


@pytest.mark.parametrize("join", [cbi.LayerKind.Add, cbi.LayerKind.Concat])
def test_joins_match_reference(gpu, join):
    """test_network.cpp:321-358: re-convergent diamond with Add / Concat."""
    rng = np.random.default_rng(50 + int(join))
    stem = conv_spec(rng, 2, cout=6, k=3, stride=1, pad=1)
    spec = cbi.NetworkSpec(2, 12, 12, [cbi.LayerDesc(cbi.LayerKind.Conv, "stem", [], stem, True)])
    for nm, cout in (("left", 4), ("right", 4 if join == cbi.LayerKind.Add else 5)):
        spec.layers.append(cbi.LayerDesc(cbi.LayerKind.Conv, nm, ["stem"],
                                         conv_spec(rng, 6, cout=cout, k=3, stride=1, pad=1)))
    spec.layers.append(cbi.LayerDesc(join, "join", ["left", "right"]))
    spec.layers.append(cbi.LayerDesc(cbi.LayerKind.Conv, "head", [],
                                     conv_spec(rng, 4 if join == cbi.LayerKind.Add else 9, k=3, stride=1, pad=1)))
    frames = [rng.uniform(0, 1, (2, 12, 12)).astype(np.float32) for _ in range(5)]
    frames[3] = frames[2].copy()
    frames[3][0, 6, 6] += 1.0
    net, _ = run_pair(spec, [0.0] * 4, frames)
    # dense equivalence at tau = 0 (test_network.cpp:330-331)
    ref = oracle.RefNet(spec, [0.0] * 4)
    assert oracle.max_rel_err(net.output(), ref.dense_forward(frames[-1])) <= TOL


@pytest.mark.parametrize("seed", range(8))
def test_c1_zero_threshold_random_networks(gpu, seed):
    """acceptance C1: tau = 0 => CB output == dense output (random conv/pool chains)."""
    rng = np.random.default_rng(101 + seed)
    c, h, w = int(rng.integers(1, 4)), int(rng.integers(12, 33)), int(rng.integers(12, 33))
    spec = random_net(rng, c, h, w, int(rng.integers(2, 6)))
    nconv = sum(1 for d in spec.layers if d.kind == cbi.LayerKind.Conv)
    net = cbi.convert_to_cb(spec, [0.0] * nconv)
    ref = oracle.RefNet(spec, [0.0] * nconv)
    x = rng.uniform(0, 1, (c, h, w)).astype(np.float32)
    for t in range(6):
        got = net.forward_frame(x)
        assert oracle.max_rel_err(got, ref.dense_forward(x)) <= TOL
        x = x.copy()
        k = int(rng.integers(0, h * w // 8 + 1))
        x[:, rng.integers(0, h, k), rng.integers(0, w, k)] = rng.uniform(0, 1, (c, k)).astype(np.float32)


def test_c2_closed_loop_consistency(gpu):
    """acceptance C2: every Detect conv's retained output == conv(its input state)."""
    rng = np.random.default_rng(102)
    spec = random_net(rng, 2, 24, 28, 4)
    nconv = sum(1 for d in spec.layers if d.kind == cbi.LayerKind.Conv)
    net = cbi.convert_to_cb(spec, [float(t) for t in rng.uniform(0.005, 0.08, nconv)])
    convs = [d.conv for d in spec.layers if d.kind == cbi.LayerKind.Conv]
    x = rng.uniform(0, 1, (2, 24, 28)).astype(np.float32)
    for t in range(6):
        net.forward_frame(x)
        ci = 0
        for i, n in enumerate(net.nodes()):
            if n.kind != cbi.LayerKind.Conv:
                continue
            st = net.node_state(i)
            want = np.zeros(n.out_shape, np.float32)
            keep = []
            cs = convs[ci]._c(keep)
            oracle.ref().ref_conv2d_dense(p(st), *st.shape, C.byref(cs), p(want))
            if n.fuse_relu:
                want = np.maximum(want, 0)
            assert oracle.max_rel_err(net.node_output(i), want) <= TOL, (t, n.name)
            ci += 1
        x = (x + rng.uniform(-0.05, 0.05, x.shape) * (rng.random(x.shape) < 0.2)).astype(np.float32)


def test_clone_is_an_independent_stream(gpu):
    spec = cbi.make_small_spec(6, 2, 32, 32)
    frames = frames_for(32, 32, n=6, c=2, noise=0.01)
    a = cbi.convert_to_cb(spec, [0.02] * 3)
    for f in frames[:3]:
        a.forward_frame(f)
    b = a.clone()
    for f in frames[3:]:
        assert np.array_equal(a.forward_frame(f), b.forward_frame(f))
    b.forward_frame(frames[0])  # advancing the clone leaves the original untouched
    ya = a.output().copy()
    a.forward_frame(frames[-1])
    assert np.array_equal(a.output(), ya)


def test_pinned_seg7_full_resolution_against_reference(gpu):
    """make_seg7_spec at its pinned 776x1040 dims (crop + ceil-mode pooling):
    bootstrap + one sparse frame, layer-1 change set bit-exact."""
    spec = cbi.make_seg7_spec(1)
    frames = cbi.gen_synthetic(cbi.SyntheticConfig(776, 1040, 3, 2, 2, 24, 4, 4, 0.0, 7))
    net = cbi.convert_to_cb(spec, [0.05] * 5)
    ref = oracle.RefNet(spec, [0.05] * 5)
    for t in range(2):
        got = net.forward_frame(frames[t])
        want = ref.forward(frames[t])
        assert got.shape == (8, 136, 218)
        assert oracle.max_rel_err(got, want) <= TOL
        gm, gi = net.node_changes(0)
        assert np.array_equal(gm, ref.stats(0)["map"])
        for i in range(len(net.nodes())):
            assert len(net.node_changes(i)[1]) == ref.stats(i)["changed_px"]


def test_openpose_style_graph_cfg3(gpu):
    """BASELINE configs[2]: OpenPose-style graph (VGG front end, two-branch
    stages re-joined by Concat) at 368x368 on a moving-subject sequence, as a
    reference manifest with from= producers. Width-reduced (channels / 8, the
    38 / 19 heads kept) so the CPU reference checks it in seconds."""
    H = W = 368
    spec = cbi.make_openpose_spec(5, H, W, width_div=8, stages=2)
    n_conv = sum(1 for d in spec.layers if d.kind == cbi.LayerKind.Conv)
    taus = [0.02] * n_conv
    net = cbi.convert_to_cb(spec, taus)
    ref = oracle.RefNet(spec, taus)
    frames = cbi.gen_synthetic(cbi.SyntheticConfig(H, W, 3, 4, 1, 64, 5, 3, 0.0, 31))
    names = [n.name for n in net.nodes()]
    for t, f in enumerate(frames):
        net.forward_frame(f)
        ref.forward(f)
        assert np.array_equal(net.node_output(0), ref.output(0)), f"frame {t}: conv1_1 not bit-exact"
        agree = []
        for i, nm in enumerate(names):
            assert oracle.max_rel_err(net.node_output(i), ref.output(i)) <= 1e-4, (t, nm)
            gm, _ = net.node_changes(i)
            agree.append(float(np.mean(gm == ref.stats(i)["map"])))
        assert min(agree) >= 0.999, (t, min(agree))
    st = ref.stats(names.index("concat_stage2"))
    assert st["changed_px"] > 0  # the join saw changes


def test_yolo_style_detector_cfg4(gpu):
    """BASELINE configs[3]: tiny-YOLO-style detector (3x3 conv + pool stack, 1x1
    head of 125 maps) on a static-camera surveillance sequence with a few moving
    objects and sensor noise; width- and resolution-reduced (270x480, channels /
    8) for the CPU reference."""
    H, W = 270, 480
    spec = cbi.make_yolo_spec(9, H, W, width_div=8)
    n_conv = sum(1 for d in spec.layers if d.kind == cbi.LayerKind.Conv)
    taus = [0.03] * n_conv
    net = cbi.convert_to_cb(spec, taus)
    ref = oracle.RefNet(spec, taus)
    frames = cbi.gen_synthetic(cbi.SyntheticConfig(H, W, 3, 4, 3, 24, 4, 6, 0.002, 77))
    for t, f in enumerate(frames):
        got = net.forward_frame(f)
        want = ref.forward(f)
        assert np.array_equal(net.node_output(0), ref.output(0)), f"frame {t}: conv1 not bit-exact"
        gm, gi = net.node_changes(0)
        assert np.array_equal(gm, ref.stats(0)["map"])
        assert oracle.max_rel_err(got, want) <= 1e-4, t
        for i in range(len(net.nodes())):
            assert float(np.mean(net.node_changes(i)[0] == ref.stats(i)["map"])) >= 0.999, (t, i)


def test_stats_csv_byte_identical(gpu):
    """forward_sequence + write_stats_csv (network.cpp:505-525, io.cpp:660-672) from
    the GPU's device counts is byte-identical to the reference's CSV (timing off,
    so wall_ns is 0 on both sides); with dense references, the per-frame losses
    agree to the GEMM's accuracy and every other column is identical."""
    H, W = 96, 128
    spec = cbi.make_seg_spec(6, H, W)
    taus = [0.05] * 5
    sc = cbi.SyntheticConfig(H, W, 3, 5, 3, 10, 3, 3, 0.003, 91)
    frames = cbi.gen_synthetic(sc)
    net = cbi.convert_to_cb(spec, taus)
    got = cbi.write_stats_csv(cbi.forward_sequence(net, frames).stats)
    want = oracle.ref_seg_stats_csv(6, H, W, taus, sc)
    assert got == want
    assert got.count("\n") == 1 + 5 * 7
    ref = oracle.RefNet(spec, taus)
    dense = np.stack([ref.dense_forward(f) for f in frames])
    net.reset()
    g = cbi.write_stats_csv(cbi.forward_sequence(net, frames, dense).stats).splitlines()
    w = oracle.ref_seg_stats_csv(6, H, W, taus, sc, with_reference=True).splitlines()
    assert len(g) == len(w)
    for a, b in zip(g[1:], w[1:]):
        ga, wa = a.split(","), b.split(",")
        assert ga[:6] == wa[:6]
        assert float(ga[6]) == pytest.approx(float(wa[6]), rel=1e-3, abs=1e-8)  # mse of a <=1e-4 deviation


def _conv(name, cin, cout, k, stride, pad, relu, rng, frm=None):
    s = cbi.ConvSpec(cin, cout, k, k, stride, pad)
    a = 1.0 / np.sqrt(cin * k * k)
    s.weights = rng.uniform(-a, a, s.weight_count()).astype(np.float32)
    s.bias = rng.uniform(-0.1, 0.1, cout).astype(np.float32)
    d = cbi.LayerDesc(cbi.LayerKind.Conv, name, list(frm or []), s, relu)
    return d


@pytest.mark.parametrize("prec", ["f16", "tf32"])
def test_wide_strided_and_reused_layers(gpu, monkeypatch, prec):
    """Tensor-path corners under both operand splits: Cout 300 (two N tiles of
    256), stride-2 5x5 with padding, K > 4000 (a 9x9 over 56 channels), Cout
    40 / 24 (N tiles 64 / 32), a Reuse1x1 layer whose GEMM source is the
    producer's output (magnitude bound through amax_origin), and inputs of
    magnitude ~40 (fp16 operands need scaling)."""
    monkeypatch.setenv("CBG_GEMM_PREC", prec)
    rng = np.random.default_rng(91)
    L = [_conv("A", 3, 40, 3, 1, 1, True, rng), _conv("B", 40, 300, 5, 2, 2, True, rng),
         _conv("C", 300, 56, 1, 1, 0, True, rng), _conv("D", 56, 24, 9, 1, 4, True, rng),
         _conv("E", 24, 24, 1, 1, 0, False, rng)]
    spec = cbi.NetworkSpec(3, 44, 52, L)
    taus = [0.5, 0.05, 0.05, 0.02, 0.02]
    pol = [cbi.DetectionPolicy.Detect] * 4 + [cbi.DetectionPolicy.Reuse1x1]
    frames = 40.0 * cbi.gen_synthetic(cbi.SyntheticConfig(44, 52, 3, 5, 2, 9, 2, 3, 0.002, 17))
    run_pair(spec, taus, frames, pol)


def test_many_streams_mixed_activity(gpu):
    """33 streams in one set (odd count, not a multiple of the GEMM grid's
    structure), some static, some with motion, some after a reset."""
    S, H, W = 33, 48, 64
    spec = cbi.make_seg_spec(7, H, W)
    taus = [0.05] * 5
    seqs = []
    for s in range(S):
        n_obj = 0 if s % 3 == 0 else (s % 5) + 1
        seqs.append(cbi.gen_synthetic(cbi.SyntheticConfig(H, W, 3, 4, n_obj, 8, 2, 2, 0.0, 50 + s)))
    net = cbi.convert_to_cb(spec, taus, n_streams=S)
    refs = [oracle.RefNet(spec, taus) for _ in range(S)]
    for t in range(4):
        if t == 2:
            net.reset(5)
            refs[5].reset()
        net.enqueue(np.stack([seqs[s][t] for s in range(S)]))
        counts = net.counts()
        for s in range(S):
            want = refs[s].forward(seqs[s][t])
            assert oracle.max_rel_err(net.output(s), want) <= TOL, (t, s)
            assert counts[0, s] == refs[s].stats(0)["changed_px"], (t, s)


def test_odd_resolution_scalar_ingest_paths(gpu):
    """H*W not a multiple of 4: the frame-ingest detect falls back to its scalar
    kernels (fp32 CHW state and 8-bit PNM ingest); results still match the
    reference, the first layer bit-exact."""
    H, W = 63, 85
    spec = cbi.make_seg_spec(8, H, W)
    taus = [0.05] * 5
    raw = cbi.gen_synthetic(cbi.SyntheticConfig(H, W, 3, 4, 2, 9, 2, 3, 0.01, 33))
    pnm = cbi.to_pnm8(raw)
    f32 = cbi.from_pnm8(pnm)
    a = cbi.convert_to_cb(spec, taus)
    b = cbi.convert_to_cb(spec, taus)
    ref = oracle.RefNet(spec, taus)
    for t in range(len(raw)):
        a.forward_frame(f32[t])
        b.forward_frame_u8(pnm[t])
        want = ref.forward(f32[t])
        assert np.array_equal(a.output(), b.output())
        assert np.array_equal(a.node_output(0), ref.output(0))
        assert oracle.max_rel_err(a.output(), want) <= TOL


@pytest.mark.parametrize("direct", ["0", "1"])
def test_a_operand_paths(gpu, monkeypatch, direct):
    """Both producers of the tcgen05 A operand (direct global->TMEM, the default;
    shared-memory staging with fetch warps, CBG_GEMM_DIRECT=0) on the seg net."""
    monkeypatch.setenv("CBG_GEMM_DIRECT", direct)
    spec = cbi.make_seg_spec(9, 80, 112)
    run_pair(spec, [0.05] * 5, frames_for(80, 112, noise=0.003))


def test_tma_gather4_a_path_for_1x1_layers(gpu, monkeypatch):
    """The experimental A producer of 1x1 layers (CBG_TMA_1X1=1): the tile's rows
    arrive by TMA tile::gather4 into the staged path's swizzled stages (DESIGN.md
    §8.25; slower than the direct path, kept off by default)."""
    monkeypatch.setenv("CBG_TMA_1X1", "1")
    spec = cbi.make_seg_spec(9, 80, 112)
    run_pair(spec, [0.05] * 5, frames_for(80, 112, noise=0.003))


def test_detached_output_copy_pipelines(gpu):
    """cbg_net_copy_output_detached: frame k's output lands in its own host
    buffer although frame k+1 (and k+2) were enqueued before anyone waited;
    the bytes equal the synchronous readback of a twin network."""
    S, H, W, T = 2, 40, 56, 5
    spec = cbi.make_seg_spec(6, H, W)
    frames = np.stack([cbi.gen_synthetic(cbi.SyntheticConfig(H, W, 3, T, 2, 8, 2, 2, 0.01, 40 + s))
                       for s in range(S)], axis=1)
    a = cbi.convert_to_cb(spec, [0.03] * 5, n_streams=S)
    b = cbi.convert_to_cb(spec, [0.03] * 5, n_streams=S)
    nbytes = a.output_bytes(-1)
    bufs = [np.zeros(nbytes // 4, np.float32) for _ in range(T)]
    want = []
    for t in range(T):
        a.enqueue(frames[t])
        a.copy_output_detached(bufs[t].ctypes.data)
        b.enqueue(frames[t])
        w = np.zeros(nbytes // 4, np.float32)
        b.copy_output_async(w.ctypes.data)
        b.synchronize()
        want.append(w)
    a.synchronize()
    for t in range(T):
        assert np.array_equal(bufs[t], want[t]), t


def test_output_delta_mirror_equals_full_output(gpu):
    """cbg_net_copy_output_delta + cbg_net_apply_output_delta: a host mirror kept
    from the per-frame deltas (changed pixels + their output vectors only) equals
    the full raw output (copy_output_async) after every frame, with frames
    enqueued back to back (two host buffers alternating), through a full update
    (reset of one stream), a tau change and a forced full frame — larger than the
    DMA estimate from the recent deltas, so its tail takes the overflow path."""
    S, H, W, T = 3, 240, 320, 9
    spec = cbi.make_seg_spec(8, H, W)
    frames = np.stack([cbi.gen_synthetic(cbi.SyntheticConfig(H, W, 3, T, 2, 10, 2, 3, 0.01, 70 + s))
                       for s in range(S)], axis=1)
    net = cbi.convert_to_cb(spec, [0.03] * 5, n_streams=S)
    nbytes = net.output_bytes(-1)
    bufs = [cbi.HostBuffer(net.output_delta_bytes(-1)) for _ in range(2)]
    mirror = np.zeros(nbytes // 4, np.float32)
    full = cbi.HostBuffer(nbytes, np.float32)
    pending = None
    for t in range(T):
        if t == 4:
            net.reset(1)
        if t == 6:
            net.set_thresholds([0.02] * 5)
        net.enqueue(frames[t], flags=_lib.FWD_FORCE_FULL if t == 7 else 0)
        net.copy_output_delta(bufs[t % 2].ptr)
        dma = net.last_delta_dma_bytes()
        if pending is not None:  # the previous frame's delta, applied while this frame runs
            net.apply_output_delta(bufs[pending % 2].ptr, mirror.ctypes.data)
            np.testing.assert_array_equal(mirror, want, err_msg=f"frame {pending}")
        net.copy_output_async(full.ptr)
        net.synchronize()
        want = full.array.copy()
        n = net.delta_counts(bufs[t % 2].array)
        cnt = net.counts()[-1]
        assert np.array_equal(n, cnt), (t, n, cnt)
        used = 16 + sum((4 * int(k) + 15) // 16 * 16 + 32 * int(k) for k in n)  # Cs = 8
        if t == 7:
            assert used > dma, (used, dma)  # the forced full frame overflowed the estimate
        pending = t
    net.apply_output_delta(bufs[pending % 2].ptr, mirror.ctypes.data, streams=(0, 2))
    net.apply_output_delta(bufs[pending % 2].ptr, mirror.ctypes.data, streams=(2, 3))
    np.testing.assert_array_equal(mirror, want)


def test_output_delta_applied_on_another_thread(gpu):
    """The e2e loop's pattern (bench.py run_e2e): frames and delta copies are
    enqueued on one host thread while a background thread applies frame k - LAG
    into the mirror; a host buffer is handed to a new copy only after its apply
    returned (cbg.h). After the last apply the mirror equals the full output."""
    from concurrent.futures import ThreadPoolExecutor
    S, H, W, T, LAG = 4, 120, 160, 12, 2
    spec = cbi.make_seg_spec(8, H, W)
    frames = np.stack([cbi.gen_synthetic(cbi.SyntheticConfig(H, W, 3, T, 3, 12, 3, 4, 0.01, 90 + s))
                       for s in range(S)], axis=1)
    net = cbi.convert_to_cb(spec, [0.03] * 5, n_streams=S)
    nbytes = net.output_bytes(-1)
    bufs = [cbi.HostBuffer(net.output_delta_bytes(-1)) for _ in range(LAG + 1)]
    mirror = np.zeros(nbytes // 4, np.float32)
    pool = ThreadPoolExecutor(max_workers=1)
    pending = {}
    apply = lambda k: net.apply_output_delta(bufs[k % (LAG + 1)].ptr, mirror.ctypes.data)
    for t in range(T):
        if (t - LAG - 1) in pending:
            pending.pop(t - LAG - 1).result()
        net.enqueue(frames[t])
        net.copy_output_delta(bufs[t % (LAG + 1)].ptr)
        if t >= LAG:
            pending[t - LAG] = pool.submit(apply, t - LAG)
    for k in sorted(pending):
        pending.pop(k).result()
    for k in range(T - LAG, T):
        apply(k)
    pool.shutdown()
    full = cbi.HostBuffer(nbytes, np.float32)
    net.copy_output_async(full.ptr)
    net.synchronize()
    np.testing.assert_array_equal(mirror, full.array)


@pytest.mark.parametrize("h,w,wd", [(1080, 1920, 8), (270, 480, 1)])
def test_yolov3_leaky_upsample_against_port(gpu, h, w, wd):
    """BASELINE configs[3] with the features the reference lacks (network.hpp:10,
    PAPER.md:647): the tiny-YOLOv3 graph — leaky ReLU (slope 0.1) on every conv,
    a x2 nearest upsampling concatenated with the 1/16 features, two heads —
    checked against the C restatement's extension (oracle/cbi_oracle.c; parity
    unpinned against the reference itself, which cannot run it). Full frame at
    channels / 8, and full width at quarter resolution. conv1 (Cout <= 16) runs
    the CUDA-core path: its leaky output is bit-exact; every map agrees."""
    spec = cbi.make_yolov3_spec(9, h, w, width_div=wd)
    n_conv = sum(1 for d in spec.layers if d.kind == cbi.LayerKind.Conv)
    taus = [0.03] * n_conv
    net = cbi.convert_to_cb(spec, taus)
    ref = oracle.PortNet(spec, taus)
    raw = cbi.gen_synthetic(cbi.SyntheticConfig(h, w, 3, 4, 3, 48, 4, 6, 0.002, 77))
    frames = cbi.from_pnm8(cbi.to_pnm8(raw))
    names = [n.name for n in net.nodes()]
    assert "up" in names and any(n.kind == cbi.LayerKind.Upsample for n in net.nodes())
    for t, f in enumerate(frames):
        got = net.forward_frame(f)
        want = ref.forward(f)
        assert np.array_equal(net.node_output(0), ref.output(0)), f"frame {t}: conv1 (leaky) not bit-exact"
        gm, gi = net.node_changes(0)
        wm, wi = ref.changes(0)
        assert np.array_equal(gm, wm) and np.array_equal(gi, wi), f"frame {t}: layer-1 map / list"
        up = names.index("up")
        assert np.array_equal(net.node_output(up), ref.output(up)) or \
            oracle.max_rel_err(net.node_output(up), ref.output(up)) <= 3e-4, t
        for i, nm in enumerate(names):
            assert float(np.mean(net.node_changes(i)[0] == ref.changes(i)[0])) >= 0.999, (t, nm)
            assert oracle.max_rel_err(net.node_output(i), ref.output(i)) <= 3e-4, (t, nm)
        assert oracle.max_rel_err(got, want) <= 3e-4, t
    assert len(net.node_changes(names.index("up"))[1]) > 0
