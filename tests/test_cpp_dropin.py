"""The C++ drop-in header (include/cbg/cbi_gpu.hpp).

CPU: it compiles standalone against include/cbg.h (C++17 and C++20).
GPU: tests/_build/dropin_parity — the header used like the reference API next
to the unmodified reference (namespace cbi) on identical frames.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "_build", "dropin_parity")


@pytest.mark.parametrize("std", ["c++17", "c++20"])
def test_header_compiles_standalone(tmp_path, std):
    src = tmp_path / "use.cpp"
    src.write_text('#include "cbg/cbi_gpu.hpp"\n'
                   "int main() { cbg::Tensor3 t(1, 2, 2); cbg::ConvSpec s; (void)s; return (int)t.size() - 4; }\n")
    r = subprocess.run(["g++", f"-std={std}", "-Wall", "-Werror", "-fsyntax-only", "-I", os.path.join(ROOT, "include"),
                        str(src)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


@pytest.mark.gpu
def test_dropin_parity_binary(gpu):
    if not os.path.exists(BIN):
        pytest.skip("tests/_build/dropin_parity not built (needs the reference headers at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASS" in r.stdout
