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


def test_quantize_rows_closed_forms():
    """R29 per-row scaling: a row whose amax is 448 has s = 1 and keeps its (e4m3-exact)
    values; a zero row has s = 1 and all-zero codes; scaling a row by 2^k scales only s; a
    row whose amax / 448 is not a power of two gets the next power of two up (amax 300 ->
    s = 1, amax 449 -> s = 2)."""
    from oracle import dit_fp8
    row = np.array([448.0, -224.0, 1.0, -3.5, 0.0, 0.015625], dtype=np.float64)  # all e4m3 values
    q, s = dit_fp8.quantize_rows(np.stack([row, np.zeros(6), row * 2.0 ** -7]))
    assert s[0] == np.float32(1.0) and s[1] == np.float32(1.0) and s[2] == np.float32(2.0 ** -7)
    assert np.array_equal(fp8.e4m3_decode(q[0]), row)
    assert np.all(q[1] == 0)
    assert np.array_equal(q[2], q[0])
    assert np.array_equal(dit_fp8.act(row[None]), row[None])
    _, s2 = dit_fp8.quantize_rows(np.array([[300.0, -1.0], [449.0, 2.0], [3.0 * 2.0 ** -20, 0.0]]))
    assert s2[0] == np.float32(1.0) and s2[1] == np.float32(2.0)
    assert s2[2] == np.float32(2.0 ** -27)  # 3 * 2^-20 / 448 = 2^-27.2 -> 2^-27


def test_fp8_block_wiring_reduces_to_the_bf16_block():
    """block(..., q8) with identity quantisers is dit.block exactly: the FP8 mode changes the
    composition only at the three R29 GEMM inputs.  With the real quantisers the block
    differs from the bf16 one by an amount of the order of e4m3's relative step (2^-4)."""
    from oracle import dit, dit_fp8
    from oracle import params as OP
    from synth import inputs
    from synth.configs import TINY
    cfg = TINY
    P = OP.Params(cfg, 0)
    r = inputs.residual(cfg, 3).astype(np.float64)
    rr = np.random.default_rng(1)
    kv = (rr.standard_normal((cfg.L_txt, cfg.d)), rr.standard_normal((cfg.L_txt, cfg.d)))
    e6 = rr.standard_normal((6, cfg.d)) * 0.1
    pos = dit.token_positions(cfg)
    ref = dit.block(P, cfg, 0, r, e6, kv, pos)
    ident = dit_fp8.Q8(act_fn=lambda h: h, weight_fn=lambda w: w)
    assert np.array_equal(dit.block(P, cfg, 0, r, e6, kv, pos, q8=ident), ref)
    got = dit.block(P, cfg, 0, r, e6, kv, pos, q8=dit_fp8.Q8())
    rel = np.linalg.norm((got - r) - (ref - r)) / np.linalg.norm(ref - r)
    assert 1e-3 < rel < 0.2, rel
