"""GPU parity at the sizes whose throughput is reported (BASELINE configs 2-5),
against the unmodified reference (oracle/_ref) run one stream per host thread,
plus the fp64 anchor (tests/fullsize.py).

What is asserted, per config (2 streams, 3-6 frames):
  * layer 1: change maps and index lists bit-exact on every frame (SURVEY.md
    §8c), and its retained output too when it runs the CUDA-core path (Cout <= 16);
  * every node: change-map disagreement with the reference <= 1% of its pixels.
    The GPU's sums differ from the reference's sequential fp32 sums by rounding
    (below), so a value within ~1e-5 of tau can be detected on one side only;
    the state then differs at that pixel until it changes again. The observed
    disagreements (profiles/r02_parity.json) are single crossings dilated by the
    downstream kernels: 0-0.33% of a node's pixels;
  * final map max_rel_err (tests/oracles.hpp:59-66) <= TOL_FINAL on every frame
    whose history is crossing-free (2x the observed maxima);
  * fp64 anchor, per closed-loop Detect conv, independent of crossings: each
    side's retained output against a float64 convolution of its own state. The
    GPU's error is bounded by ANCHOR_RATIO x the reference's and by ANCHOR_ABS.
    The ratio is not ~1: the tcgen05 fp32 accumulator truncates at every MMA
    (3 per 16 K of the 3xFP16 product), a biased error growing with K, where the
    reference's sequential fp32 sum rounds to nearest (a random walk). Measured:
    1.0x (layer 1, bit-exact), 1.1-4.4x on the seg net, up to 11x for the
    K = 9000 stage-2 convs of cfg3 (DESIGN.md §3.4 "Precision").
"""
import numpy as np
import pytest

from paper_1808_05488_b200 import cbi
from tests import fullsize

pytestmark = pytest.mark.gpu

ANCHOR_RATIO = 16.0
ANCHOR_ABS = 2.5e-4


def pnm_seq(h, w, n, objects, size, vy, vx, noise, seed):
    raw = cbi.gen_synthetic(cbi.SyntheticConfig(h, w, 3, n, objects, size, vy, vx, noise, seed))
    return cbi.from_pnm8(cbi.to_pnm8(raw))


def check(spec, taus, streams, n, tol_final):
    rep = fullsize.run_parity(spec, taus, streams, n, anchor_frames=(0, -1), anchor_streams=(0, 1))
    clean = True
    for fr in rep["per_frame"]:
        t = fr["frame"]
        assert fr["l1_bit_exact"], f"frame {t}: layer-1 map / list not bit-exact"
        if spec.layers[0].conv.out_channels <= 16:  # CUDA-core path, reference summation order
            assert fr["max_rel_err"][rep["nodes"][0]] == 0.0, f"frame {t}: layer-1 output not bit-exact"
        for name, ag in fr["agree"].items():
            assert ag >= 0.99, (t, name, ag)
        clean = clean and all(a == 1.0 for a in fr["agree"].values())
        if clean:
            assert fr["final_max_rel_err"] <= tol_final, (t, fr["final_max_rel_err"])
        for name, a in fr["anchor"].items():
            assert a["gpu_vs_fp64"] <= max(ANCHOR_RATIO * a["ref_vs_fp64"], 1e-6), (t, name, a)
            assert a["gpu_vs_fp64"] <= ANCHOR_ABS, (t, name, a)
    return rep


def test_cfg2_bench_workload_640x480(gpu):
    """The bench workload: seg net 640x480, 8-bit frames, 6 objects x 40 px, streams 1000/1001."""
    streams = [pnm_seq(480, 640, 6, 6, 40, 4, 4, 0.0, 1000 + s) for s in range(2)]
    check(cbi.make_seg_spec(1, 480, 640), [0.05] * 5, streams, 6, tol_final=6.5e-5)


def test_cfg3_openpose_full_width(gpu):
    """OpenPose-style graph at full width (VGG-19 front end, 2 stages, Concat joins), 368x368."""
    spec = cbi.make_openpose_spec(5, 368, 368, width_div=1, stages=2)
    nc = sum(1 for d in spec.layers if d.kind == cbi.LayerKind.Conv)
    streams = [pnm_seq(368, 368, 3, 1, 64, 5, 3, 0.0, 31 + s) for s in range(2)]
    check(spec, [0.02] * nc, streams, 3, tol_final=8e-4)


def test_cfg4_yolo_full_width_1080p(gpu):
    """tiny-YOLO-style detector at full width on 1920x1080 frames with sensor noise."""
    spec = cbi.make_yolo_spec(9, 1080, 1920)
    nc = sum(1 for d in spec.layers if d.kind == cbi.LayerKind.Conv)
    streams = [pnm_seq(1080, 1920, 3, 3, 48, 4, 6, 0.002, 77 + s) for s in range(2)]
    check(spec, [0.03] * nc, streams, 3, tol_final=3e-4)


def test_cfg5_seg_net_1080p(gpu):
    """The scene-labeling net at 1920x1080, streams 1000/1001 of the cfg5 stream set."""
    streams = [pnm_seq(1080, 1920, 3, 6, 40, 4, 4, 0.0, 1000 + s) for s in range(2)]
    check(cbi.make_seg_spec(1, 1080, 1920), [0.05] * 5, streams, 3, tol_final=7e-5)
