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
    ident = dit_fp8.Q8(act_fn=lambda h: h, weight_fn=lambda w: w, qk_fn=lambda x, s: x, v_fn=lambda v: v)
    assert np.array_equal(dit.block(P, cfg, 0, r, e6, kv, pos, q8=ident), ref)
    got = dit.block(P, cfg, 0, r, e6, kv, pos, q8=dit_fp8.Q8())
    rel = np.linalg.norm((got - r) - (ref - r)) / np.linalg.norm(ref - r)
    assert 1e-3 < rel < 0.2, rel


# ---------------------------------------------------------------- MXFP8 (R30): OCP MX v1.0
def test_mx_block_exponent_closed_form():
    """e = floor(log2 amax) - 8 for E4M3 elements, stored as e + 127."""
    for k in (-20, -3, 0, 1, 7, 30):
        for mant in (1.0, 1.5, 1.75, 1.99):
            x = np.zeros((1, 32))
            x[0, 5] = mant * 2.0 ** k
            x[0, 6] = -0.25 * 2.0 ** k
            _, s = fp8.mx_quantize(x)
            assert s[0, 0] == k - 8 + 127


def test_mx_worked_block_1_to_32():
    """x = 1..32: amax 32 -> e = 5 - 8 = -3, X = 1/8, x/X = 8, 16, ..., 256.  Every multiple of
    8 up to 128 is exact in e4m3 except the ones needing a 4th mantissa bit; 136 = 1.0625 * 128
    is the midpoint of 128 and 144 and rounds to even (128); 152, between 144 and 160, to 160."""
    x = np.arange(1, 33, dtype=np.float64)[None, :]
    q, s = fp8.mx_quantize(x)
    assert s[0, 0] == 124
    got = fp8.mx_dequantize(q, s)[0]
    assert got[0] == 1.0 and got[15] == 16.0 and got[31] == 32.0
    assert got[16] == 16.0          # 17 -> 136 -> 128 (tie to even) -> 16
    assert got[18] == 20.0          # 19 -> 152: midpoint of 144 and 160 -> 160 (even) -> 20
    assert got[2] == 3.0 and got[6] == 7.0   # 24 = 1.5*16, 56 = 1.75*32: exact


def test_mx_representable_blocks_round_trip_exactly():
    r = np.random.default_rng(1)
    codes = r.integers(0, 0x7F, size=(4, 64)).astype(np.uint8)  # finite, non-negative e4m3
    codes[:, ::32] = 0x70                                          # amax 256 = 2^8 in every block
    vals = fp8.e4m3_decode(codes) * np.where(r.random((4, 64)) < 0.5, -1.0, 1.0)
    scale = np.exp2(r.integers(-40, 40, size=(4, 2)))[..., None]
    x = (vals.reshape(4, 2, 32) * scale).reshape(4, 64)
    q, s = fp8.mx_quantize(x)
    np.testing.assert_array_equal(fp8.mx_dequantize(q, s), x)


def test_mx_saturation_per_ocp():
    """amax = 1.9 * 2^k: X = 2^(k-8), amax / X = 486.4 > 448 -> the code saturates at 448."""
    x = np.zeros((1, 32))
    x[0, 0] = 1.9 * 2.0 ** 3
    x[0, 1] = -1.9 * 2.0 ** 3
    x[0, 2] = 1.0
    q, s = fp8.mx_quantize(x)
    assert q[0, 0] == 0x7E and q[0, 1] == 0xFE
    d = fp8.mx_dequantize(q, s)[0]
    assert d[0] == 1.75 * 2.0 ** 3 and d[2] == 1.0


def test_mx_blocks_are_independent_and_zero_block():
    r = np.random.default_rng(2)
    x = r.standard_normal((3, 128))
    q0, s0 = fp8.mx_quantize(x)
    x2 = x.copy()
    x2[:, 32:64] *= 1000.0
    x2[1, 96:128] = 0.0
    q1, s1 = fp8.mx_quantize(x2)
    keep = np.r_[0:32, 64:128]
    np.testing.assert_array_equal(q0[0, keep], q1[0, keep])
    np.testing.assert_array_equal(q0[:, 0:32], q1[:, 0:32])
    assert s1[1, 3] == 0 and not q1[1, 96:].any()
    assert (s1[:, 1] - s0[:, 1] >= 9).all()  # 1000 ~ 2^9.97: the block exponent moved up


def test_mx_codes_match_torch_cast_of_scaled_values():
    torch = pytest.importorskip("torch")
    r = np.random.default_rng(3)
    x = (r.standard_normal((8, 256)) * np.exp2(r.integers(-10, 10, size=(8, 1)))).astype(np.float32)
    q, s = fp8.mx_quantize(x)
    scaled = x.astype(np.float64).reshape(8, 8, 32) / np.exp2(s.astype(np.float64) - 127)[..., None]
    assert np.abs(scaled).max() <= 512
    t = torch.from_numpy(np.clip(scaled, -448, 448).reshape(8, 256)).to(torch.float8_e4m3fn)
    np.testing.assert_array_equal(q, t.view(torch.uint8).numpy())


def test_mx_relative_error_bound():
    """Unsaturated normal-range elements lose at most half a quantum: |dq - x| <= 2^-4 |x|."""
    r = np.random.default_rng(4)
    x = r.standard_normal((16, 256)) * 3.0
    q, s = fp8.mx_quantize(x)
    d = fp8.mx_dequantize(q, s)
    X = np.repeat(np.exp2(s.astype(np.float64) - 127), 32, axis=1)
    ok = (np.abs(x) / X >= 2.0 ** -6) & (np.abs(x) / X <= 448)
    assert ok.mean() > 0.9
    assert (np.abs(d - x)[ok] <= 2.0 ** -4 * np.abs(x)[ok] + 1e-300).all()


def test_gemm_mxf8_bruteforce():
    r = np.random.default_rng(5)
    a = r.standard_normal((3, 64))
    b = r.standard_normal((4, 64)) * 10
    qa, sa = fp8.mx_quantize(a)
    qb, sb = fp8.mx_quantize(b)
    want = np.zeros((3, 4))
    for i in range(3):
        for j in range(4):
            acc = 0.0
            for k in range(64):
                acc += (fp8.e4m3_decode(qa[i, k:k + 1])[0] * 2.0 ** (int(sa[i, k // 32]) - 127)) * \
                       (fp8.e4m3_decode(qb[j, k:k + 1])[0] * 2.0 ** (int(sb[j, k // 32]) - 127))
            want[i, j] = acc
    np.testing.assert_allclose(fp8.gemm_mxf8(qa, sa, qb, sb), want, rtol=1e-13, atol=1e-12)


def test_mx_weight_blocks_run_along_k_per_output_column():
    """R31: W [K, N] is block-quantised along K for each output column.  Scaling column j by 2^k
    must scale exactly that column of the dequantised weight (per-tensor scaling, or blocks
    along N, would change other columns' codes)."""
    from oracle import dit_fp8
    r = np.random.default_rng(7)
    W = r.standard_normal((64, 8))
    base = dit_fp8.mx_weight(W)
    W2 = W.copy()
    W2[:, 3] *= 2.0 ** 9
    got = dit_fp8.mx_weight(W2)
    want = base.copy()
    want[:, 3] *= 2.0 ** 9
    np.testing.assert_array_equal(got, want)
    # blocks are 32 long along K: a spike in rows 0..31 of column 5 leaves rows 32..63 alone
    W3 = W.copy()
    W3[0, 5] = 1e4
    got3 = dit_fp8.mx_weight(W3)
    np.testing.assert_array_equal(got3[32:, 5], base[32:, 5])
    assert not np.array_equal(got3[1:32, 5], base[1:32, 5])


def test_mx_act_rounds_to_fp32_then_blocks_rows():
    from oracle import dit_fp8
    r = np.random.default_rng(8)
    h = r.standard_normal((3, 64)) * 3
    h[1] *= 2.0 ** 20  # rows are independent
    got = dit_fp8.mx_act(h)
    q, s = fp8.mx_quantize(h.astype(np.float32).astype(np.float64))
    np.testing.assert_array_equal(got, fp8.mx_dequantize(q, s))
    np.testing.assert_array_equal(dit_fp8.mx_act(h[[0]]), got[[0]])


def test_qk_scale_bounds_every_component_and_is_a_power_of_two():
    """R32: after the per-head RMSNorm, the gain and RoPE, every component of Q is at most
    sqrt(dh) max|g|; the worst case (all of a head's energy in one component, at the largest
    gain) lands exactly at or below 448 after dividing by qk_scale -- never saturated."""
    from oracle import dit, dit_fp8
    dh = 128
    r = np.random.default_rng(3)
    g = r.uniform(0.5, 1.5, size=dh)
    s = float(dit_fp8.qk_scale(g, dh))
    assert s > 0 and np.log2(s) == np.round(np.log2(s))
    x = np.zeros((1, dh))
    x[0, int(np.argmax(g))] = 1.0
    worst = dit.rms_norm(x, 1e-6) * g               # sqrt(dh) * max|g| in one component
    assert worst.max() / s <= 448.0
    assert worst.max() / s > 448.0 / 2              # the scale is the tightest power of two
    q = dit_fp8.qk_quant(worst, s)
    assert abs(q.max() - worst.max()) <= 2.0 ** -4 * worst.max()
    # a typical head vector keeps e4m3's relative precision (no subnormal codes)
    v = dit.rms_norm(r.standard_normal((64, dh)), 1e-6) * g
    qv = dit_fp8.qk_quant(v, s)
    big = np.abs(v) > 0.05
    assert (np.abs(qv - v)[big] <= 2.0 ** -4 * np.abs(v)[big] + 2.0 ** -8 * np.abs(v)[big]).all()


def test_v_quant_per_tensor_power_of_two():
    """R33: one power-of-two scale for the whole V: values that are e4m3 codes times the scale
    the amax implies (amax 56 = 448 / 8 -> s = 1/8) come back exactly; otherwise every element
    within e4m3's normal range keeps half-a-quantum relative precision."""
    from oracle import dit_fp8
    r = np.random.default_rng(5)
    v = r.standard_normal((64, 256))
    q = dit_fp8.v_quant(v)
    codes = fp8.e4m3_encode(np.array([1.0, -2.5, 448.0, 0.125]))
    vals = fp8.e4m3_decode(codes)[None, :] * 2.0 ** -3
    np.testing.assert_array_equal(dit_fp8.v_quant(vals), vals)   # amax 56 = 448 / 8: s = 1/8
    big = np.abs(v) > 0.5
    assert (np.abs(q - v)[big] <= 2.0 ** -4 * np.abs(v)[big] + 2.0 ** -8).all()
    # the scale is a power of two: amax 100 -> s = 2^-2 (not 100 / 448), 100 / s = 400 is the
    # midpoint of 384 and 416 and rounds to even (384): the amax comes back as 96, not 100
    w = np.array([[100.0, 1.0, -3.0]])
    assert dit_fp8.v_quant(w)[0, 0] == 96.0
