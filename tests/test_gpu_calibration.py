"""GPU-backed threshold calibration (calibration.cpp:95-180) vs the reference's
own select_thresholds / sweep_threshold_factor on the same sequences and
reference outputs. The GPU version replays every candidate of a layer at once
(one stream per candidate); selections, caps and the trace must agree."""
import numpy as np
import pytest

from paper_1808_05488_b200 import cbi
from tests import oracle

pytestmark = pytest.mark.gpu


def sequences(spec, ref, n_seq=2, n_frames=5, seed=3, labels=False):
    seqs = []
    for q in range(n_seq):
        f = cbi.gen_synthetic(cbi.SyntheticConfig(spec.in_height, spec.in_width, spec.in_channels, n_frames, 2, 6,
                                                  2, 1, 0.01, seed + q))
        r = np.stack([ref.dense_forward(x) for x in f])
        if labels:
            r = np.argmax(r, axis=1)[:, None].astype(np.float32)
        seqs.append(cbi.EvalSequence(f, r))
    return seqs


def test_select_thresholds_matches_reference(gpu):
    spec = cbi.make_small_spec(11, 2, 24, 28)
    taus0 = [0.0] * 3
    net = cbi.convert_to_cb(spec, taus0)
    ref = oracle.RefNet(spec, taus0)
    seqs = sequences(spec, ref)
    cfg = cbi.CalibConfig(initial_tau=0.004, growth_factor=1.6, per_layer_budget=2e-4, max_steps=12)
    got = cbi.select_thresholds(net, seqs, cfg)
    want = ref.select_thresholds(seqs, cfg)
    assert got.taus == want.taus
    assert got.hit_cap == want.hit_cap
    assert [(t.layer, t.tau) for t in got.trace] == [(t.layer, t.tau) for t in want.trace]
    for g, w in zip(got.trace, want.trace):
        assert g.loss == pytest.approx(w.loss, rel=1e-3, abs=1e-9)
    assert any(t > 0 for t in got.taus)


def test_select_thresholds_pixel_accuracy_worst_and_overrides(gpu):
    spec = cbi.make_small_spec(12, 2, 20, 20)
    net = cbi.convert_to_cb(spec, [0.0] * 3)
    ref = oracle.RefNet(spec, [0.0] * 3)
    seqs = sequences(spec, ref, n_seq=3, seed=40, labels=True)
    cfg = cbi.CalibConfig(initial_tau=0.01, growth_factor=2.0, budget_overrides=[0.0, 0.01, 0.05],
                          metric=cbi.LossMetric.PixelAccuracyDelta, aggregation=cbi.LossAggregation.Worst, max_steps=8)
    got = cbi.select_thresholds(net, seqs, cfg)
    want = ref.select_thresholds(seqs, cfg)
    assert got.taus == want.taus and got.hit_cap == want.hit_cap
    assert [(t.layer, t.tau, t.loss) for t in got.trace] == [(t.layer, t.tau, t.loss) for t in want.trace]


def test_sweep_threshold_factor_matches_reference(gpu):
    spec = cbi.make_small_spec(13, 2, 24, 24)
    base = [0.02, 0.03, 0.01]
    net = cbi.convert_to_cb(spec, base)
    ref = oracle.RefNet(spec, base)
    seqs = sequences(spec, ref, n_seq=2, n_frames=6, seed=70)
    factors = [0.0, 0.5, 1.0, 2.0, 4.0]
    got = cbi.sweep_threshold_factor(net, base, factors, seqs)
    want = ref.sweep_threshold_factor(base, factors, seqs)
    for g, w in zip(got, want):
        assert g.factor == w.factor
        assert g.loss == pytest.approx(w.loss, rel=1e-3, abs=1e-9)
        assert g.total_eff_ops == w.total_eff_ops
    assert got[0].loss == pytest.approx(0.0, abs=1e-9)  # factor 0 = tau 0 = the dense output
    assert got[-1].total_eff_ops < got[0].total_eff_ops


def test_calibration_argument_errors(gpu):
    spec = cbi.make_small_spec(14, 2, 16, 16)
    net = cbi.convert_to_cb(spec, [0.0] * 3)
    ref = oracle.RefNet(spec, [0.0] * 3)
    seqs = sequences(spec, ref, n_seq=1, n_frames=2)
    with pytest.raises(cbi.InvalidInputError):
        cbi.select_thresholds(net, seqs, cbi.CalibConfig(initial_tau=0.0))
    with pytest.raises(cbi.InvalidInputError):
        cbi.select_thresholds(net, seqs, cbi.CalibConfig(growth_factor=1.0))
    with pytest.raises(cbi.InvalidInputError):
        cbi.select_thresholds(net, seqs, cbi.CalibConfig(budget_overrides=[0.1]))
    with pytest.raises(cbi.InvalidInputError):
        cbi.sweep_threshold_factor(net, [0.1] * 3, [1.0, 0.5], seqs)
    with pytest.raises(cbi.InvalidInputError):
        cbi.sweep_threshold_factor(net, [0.1] * 2, [1.0], seqs)


def test_per_stream_thresholds(gpu):
    """A stream set with different thresholds per stream == separate networks."""
    spec = cbi.make_small_spec(15, 2, 20, 24)
    frames = cbi.gen_synthetic(cbi.SyntheticConfig(20, 24, 2, 5, 2, 5, 1, 2, 0.02, 5))
    taus = [[0.0, 0.0, 0.0], [0.02, 0.05, 0.01], [0.1, 0.0, 0.2]]
    net = cbi.convert_to_cb(spec, [0.0] * 3, n_streams=3)
    for s, t in enumerate(taus):
        net.set_stream_thresholds(s, t)
    refs = [oracle.RefNet(spec, t) for t in taus]
    for f in frames:
        net.enqueue(np.stack([f] * 3))
        for s in range(3):
            want = refs[s].forward(f)
            assert oracle.max_rel_err(net.output(s), want) <= 1e-4
            assert net.counts()[0, s] == refs[s].stats(0)["changed_px"]
