"""Pins of oracle/fp8.py (NEXT-4, R28) against the E4M3 format definition, a
brute-force loop and torch's float8_e4m3fn cast (a library routine) -- CPU only."""
import numpy as np
import pytest
import torch

from oracle import fp8
from synth import inputs


def test_decode_closed_forms():
    """Format constants: 1.0 = 0x38, 448 = 0x7E (largest finite), 2^-6 = 0x08 (smallest
    normal), 2^-9 = 0x01 (smallest subnormal), 0x7F / 0xFF are NaN, 0x80 is -0."""
    d = fp8.e4m3_decode(np.array([0x38, 0x7E, 0x08, 0x01, 0x00, 0xB8, 0x07, 0x3C], dtype=np.uint8))
    assert list(d) == [1.0, 448.0, 2.0 ** -6, 2.0 ** -9, 0.0, -1.0, 7 * 2.0 ** -9, 1.5]
    assert np.isnan(fp8.e4m3_decode(np.array([0x7F, 0xFF], dtype=np.uint8))).all()
    assert np.signbit(fp8.e4m3_decode(np.array([0x80], dtype=np.uint8)))[0]


def test_round_trip_all_codes():
    codes = np.array([c for c in range(256) if c not in (0x7F, 0xFF)], dtype=np.uint8)
    assert np.array_equal(fp8.e4m3_encode(fp8.e4m3_decode(codes)), codes)


def test_ties_to_even_and_saturation():
    v = np.array([1 + 1 / 16, 1 + 3 / 16, 2.0 ** -10, 3 * 2.0 ** -10, 1000.0, -1000.0, 464.0, 447.0, -0.0],
                 dtype=np.float64)
    # 1.0625 -> 1.0 (even mantissa 0), 1.1875 -> 1.25 (even 2), 2^-10 -> 0 (even 0),
    # 3*2^-10 -> 2*2^-9 (even 2), +-1000 -> +-448, 464 (tie 448/480) -> 448, 447 -> 448
    want = [0x38, 0x3A, 0x00, 0x02, 0x7E, 0xFE, 0x7E, 0x7E, 0x80]
    assert list(fp8.e4m3_encode(v)) == want


def test_encode_matches_torch_cast_in_range():
    g = np.random.default_rng(5)
    v = np.concatenate([g.standard_normal(20000) * s for s in (1e-3, 0.05, 1.0, 30.0, 200.0)]).astype(np.float32)
    v = v[np.abs(v) <= 448]
    want = torch.from_numpy(v).to(torch.float8_e4m3fn).view(torch.uint8).numpy()
    assert np.array_equal(fp8.e4m3_encode(v), want)


def test_quantize_scale_property_and_zero():
    x = inputs.bf16_bits_to_f64(inputs.activation_bf16((64, 96), seed=3)).astype(np.float32)
    q, s = fp8.quantize_per_tensor(x)
    d = fp8.e4m3_decode(q)
    assert s == np.float32(np.abs(x).max() / np.float32(448))
    assert np.abs(d).max() == 448.0  # the amax element lands on the largest finite code
    # every element within half a quantum (relative 2^-4 normal, absolute 2^-10 * s subnormal)
    err = np.abs(d * np.float64(s) - x)
    assert np.all(err <= np.maximum(np.abs(x) * 2.0 ** -4, 2.0 ** -10 * float(s)) * 1.0001)
    q0, s0 = fp8.quantize_per_tensor(np.zeros((4, 4), np.float32))
    assert s0 == 1.0 and not q0.any()


def test_gemm_bruteforce():
    g = np.random.default_rng(1)
    qa = g.integers(0, 256, size=(3, 5)).astype(np.uint8)
    qb = g.integers(0, 256, size=(4, 5)).astype(np.uint8)
    qa[(qa & 0x7F) == 0x7F] = 0
    qb[(qb & 0x7F) == 0x7F] = 0
    out = fp8.gemm_e4m3(qa, qb, 0.5, 3.0)
    for i in range(3):
        for j in range(4):
            acc = 0.0
            for k in range(5):
                acc += fp8.e4m3_decode(qa[i, k]) * fp8.e4m3_decode(qb[j, k])
            assert out[i, j] == pytest.approx(1.5 * acc, rel=1e-12, abs=1e-300)
