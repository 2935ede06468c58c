"""GPU: the fused dilate+compact kernel vs the reference's dilate_window /
propagate_changes / extract_indexes (acceptance C3, acceptance.cpp:125-172),
bit-exact, over kernel sizes 1..7, strides 1..3 (stride 1 and 2 have bit-domain
fast paths, 3 the generic path), paddings 0..3, pinned (cropped) output dims,
and map densities from a single pixel to full. Driven through a standalone
Propagate-policy CBConvLayer (the path a propagate layer takes in a network).
"""
import ctypes as C

import numpy as np
import pytest

from paper_1808_05488_b200 import cbi
from tests import oracle
from tests.oracle import p

pytestmark = pytest.mark.gpu


def ref_dilate(m, kh, kw, s, pad, oh, ow):
    out = np.zeros((oh, ow), np.uint8)
    oracle.ref().ref_dilate_window(p(np.ascontiguousarray(m)), m.shape[0], m.shape[1], kh, kw, s, pad, oh, ow,
                                   p(out))
    return out


def cases(rng, n):
    for _ in range(n):
        h, w = int(rng.integers(1, 40)), int(rng.integers(1, 90))
        kh, kw = int(rng.integers(1, 8)), int(rng.integers(1, 8))
        s, pad = int(rng.integers(1, 4)), int(rng.integers(0, 4))
        if h + 2 * pad - kh < 0 or w + 2 * pad - kw < 0:
            continue
        oh, ow = (h + 2 * pad - kh) // s + 1, (w + 2 * pad - kw) // s + 1
        pin = rng.random() < 0.25
        if pin:  # crop (tensor.hpp:49-53)
            oh, ow = max(1, oh - int(rng.integers(0, 3))), max(1, ow - int(rng.integers(0, 3)))
        yield h, w, kh, kw, s, pad, oh, ow, pin


@pytest.mark.parametrize("density", [0.0, 0.002, 0.05, 0.3, 1.0])
def test_dilate_compact_matches_reference(gpu, density):
    rng = np.random.default_rng(int(density * 1000) + 3)
    checked = 0
    for h, w, kh, kw, s, pad, oh, ow, pin in cases(rng, 120):
        spec = cbi.ConvSpec(1, 1, kh, kw, s, pad, oh if pin else 0, ow if pin else 0,
                            np.zeros(kh * kw, np.float32), np.zeros(1, np.float32))
        layer = cbi.CBConvLayer(spec, 0.0, cbi.DetectionPolicy.Propagate, in_height=h, in_width=w)
        assert (layer.out_h, layer.out_w) == (oh, ow)
        x = np.zeros((1, h, w), np.float32)
        layer.forward(x, force_full_update=True)
        for rep in range(2):
            m = (rng.random((h, w)) < density).astype(np.uint8)
            if density == 0.002:
                m[:] = 0
                m[int(rng.integers(0, h)), int(rng.integers(0, w))] = 1
            res = layer.forward(x, cbi.UpstreamChange(m, np.argwhere(m).astype(np.int32)))
            want = ref_dilate(m, kh, kw, s, pad, oh, ow)
            assert np.array_equal(res.out_map, want), (h, w, kh, kw, s, pad, oh, ow)
            assert np.array_equal(res.indexes, np.argwhere(want).astype(np.int32))
            checked += 1
    assert checked > 100


def test_wide_maps_multiword_rows(gpu):
    """Rows spanning many 32-pixel words, multiple tiles, pool-style stride 2."""
    rng = np.random.default_rng(9)
    for (h, w, k, s, pad) in ((37, 1000, 7, 1, 3), (120, 517, 2, 2, 0), (64, 333, 3, 2, 1), (9, 2049, 1, 1, 0)):
        oh, ow = (h + 2 * pad - k) // s + 1, (w + 2 * pad - k) // s + 1
        spec = cbi.ConvSpec(1, 1, k, k, s, pad, 0, 0, np.zeros(k * k, np.float32), np.zeros(1, np.float32))
        layer = cbi.CBConvLayer(spec, 0.0, cbi.DetectionPolicy.Propagate, in_height=h, in_width=w)
        x = np.zeros((1, h, w), np.float32)
        layer.forward(x, force_full_update=True)
        m = (rng.random((h, w)) < 0.01).astype(np.uint8)
        res = layer.forward(x, cbi.UpstreamChange(m, np.argwhere(m).astype(np.int32)))
        assert np.array_equal(res.out_map, ref_dilate(m, k, k, s, pad, oh, ow))
