"""CPU check of the device 8-bit ingest arithmetic (change_kernels.cu,
detect_frame_u8_kernel): load_pnm divides each byte by 255.0f (io.cpp:389-397);
the kernel computes q = fl(v * fl(1/255)) and fl(fma(fma(-q, 255, v), fl(1/255), q)).
Every step is emulated exactly in float64 (products of two fp32 values are
exact in 53 bits; the sums here cancel or stay within 53 bits) and rounded
once to fp32, so the comparison is exact."""
import numpy as np

f32 = np.float32


def _fma32(a, b, c):
    return f32(np.float64(a) * np.float64(b) + np.float64(c))


def test_byte_div255_sequence():
    inv = f32(1.0) / f32(255.0)
    for v in range(256):
        want = np.divide(f32(v), f32(255.0), dtype=np.float32)  # IEEE correctly rounded
        q = f32(f32(v) * inv)
        got = _fma32(_fma32(-q, f32(255.0), f32(v)), inv, q)
        assert got == want, v


def test_plain_multiply_is_not_enough():
    """why the residual step exists: v * fl(1/255) misrounds about half the bytes"""
    inv = f32(1.0) / f32(255.0)
    bad = sum(f32(f32(v) * inv) != np.divide(f32(v), f32(255.0), dtype=np.float32) for v in range(256))
    assert bad > 0
