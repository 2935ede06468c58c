"""CPU: the C-ABI library loads without a GPU, exports every symbol
include/cbg.h declares, and its host-side logic (resolve + convert_to_cb
validation, error categories) mirrors the reference (network.cpp:37-133,
416-503; common.hpp:11-21). No compute calls are made here.
"""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_1808_05488_b200 import _lib, cbi
from tests import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    with open(os.path.join(ROOT, "include", "cbg.h")) as fh:
        text = fh.read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(cbg_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(_lib.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 40
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # and the Python binding declares a signature for each of them
    assert sorted(_lib.SIGNATURES) == syms


def test_abi_version_and_device_probe_without_gpu():
    assert _lib.lib.cbg_abi_version() == 1
    assert _lib.lib.cbg_device_available() in (0, 1)


def test_ctx_create_fails_loudly_without_device():
    if cbi.device_available():
        pytest.skip("a device is visible")
    with pytest.raises(_lib.UnsupportedError):
        cbi.Context(0)


def seg(seed=1):
    return cbi.make_seg_spec(seed, 64, 64)


def test_convert_validation_categories():
    spec = seg()
    cbi.validate_network(spec, [0.1] * 5)
    with pytest.raises(cbi.InvalidInputError, match="expected 5 thresholds"):
        cbi.validate_network(spec, [0.1])
    with pytest.raises(cbi.InvalidInputError, match="tau must be >= 0"):
        cbi.validate_network(spec, [0.1, -0.2, 0.1, 0.1, 0.1])
    pol = [cbi.DetectionPolicy.Propagate] + [cbi.DetectionPolicy.Detect] * 4
    with pytest.raises(cbi.ConfigError, match="propagate"):
        cbi.validate_network(spec, [0.0] * 5, pol)
    pol = [cbi.DetectionPolicy.Detect] * 3 + [cbi.DetectionPolicy.Reuse1x1] * 2
    cbi.validate_network(spec, [0.0] * 5, pol)  # L6, L7 are 1x1 (test_network.cpp:208-216)
    pol[1] = cbi.DetectionPolicy.Reuse1x1
    with pytest.raises(cbi.ConfigError, match="reuse_1x1"):
        cbi.validate_network(spec, [0.0] * 5, pol)


def test_resolve_errors_name_the_layer():
    spec = cbi.NetworkSpec(3, 16, 16, [cbi.LayerDesc(cbi.LayerKind.Conv, "bad", [], cbi.ConvSpec(4, 2, 3, 3))])
    spec.layers[0].conv.weights = np.zeros(spec.layers[0].conv.weight_count(), np.float32)
    spec.layers[0].conv.bias = np.zeros(2, np.float32)
    with pytest.raises(cbi.InvalidInputError) as e:
        cbi.validate_network(spec, [0.0])
    assert "bad" in str(e.value) and "layer 0" in str(e.value)  # test_network.cpp:59-79


def test_act_absorption_rules():
    spec = seg()
    cbi.validate_network(spec, [0.0] * 5)  # Act rows absorbed into L1/L3
    bad = cbi.NetworkSpec(3, 16, 16, [cbi.LayerDesc(cbi.LayerKind.Act, "a")])
    with pytest.raises(cbi.ConfigError, match="absorbed"):
        cbi.validate_network(bad, [])


def test_restatement_agrees_on_validation():
    """The C port raises the same categories as the product for the same specs."""
    if not oracle.port_available():
        pytest.skip("port not built")
    spec = seg()
    for taus, pol, exc in (([0.1], None, cbi.InvalidInputError),
                           ([0.0] * 5, [1, 0, 0, 0, 0], cbi.ConfigError),
                           ([0.0] * 5, [0, 2, 0, 0, 0], cbi.ConfigError)):
        with pytest.raises(exc):
            cbi.validate_network(spec, taus, pol)
        with pytest.raises(exc):
            oracle.PortNet(spec, taus, pol)
