"""fp64/fp32 CPU ORACLE for the FP8 (e4m3) GEMM of SURVEY NEXT-4.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): never imported by the product path.

PAPER.md names quantisation only as a serving optimisation of the systems it builds on
("FP8/INT8 quantisation"); it fixes no format, so this follows DESIGN.md R28:
  * the OCP FP8 E4M3 ("e4m3fn") format -- 1 sign, 4 exponent (bias 7), 3 mantissa bits,
    no infinities, S.1111.111 = NaN, largest finite 448 = 1.75 * 2^8, smallest subnormal
    2^-9; conversion rounds to nearest, ties to even, and saturates to +-448;
  * per-tensor current scaling: s = amax|x| / 448 (1 when x == 0), q = e4m3(x / s); the
    scale and the division are taken in fp32 (the kernel's precision -- a float decides an
    integer code here, so both sides decide it in the same precision, rule 3);
  * the GEMM: out = s_a * s_b * (dec(q_a) . dec(q_b)^T), exact products summed in fp64.

Parity status (pins in tests/test_oracle_fp8.py): encode/decode pinned by the format's
closed-form values, the 256-code round trip, ties-to-even midpoints, saturation and
torch's float8_e4m3fn cast (a library routine) on in-range values; quantize pinned by the
scale property (the amax element maps to 448) and the zero tensor; gemm pinned by a
brute-force loop on a tiny case.  MXFP8 (R30, below): mx_quantize pinned by the block
exponent's closed form, the worked block 1..32 (ties-to-even at 136), exact round trips of
representable blocks, OCP saturation, block independence, the zero block and torch's
float8_e4m3fn cast on the scaled values; gemm_mxf8 by a brute-force loop.
"""
import numpy as np

E4M3_MAX = 448.0


def e4m3_decode(b):
    """bytes (uint8 array) -> fp64 values (NaN for the two NaN codes)."""
    b = np.asarray(b, dtype=np.uint8).astype(np.int64)
    sign = np.where(b & 0x80, -1.0, 1.0)
    e = (b >> 3) & 0xF
    m = b & 0x7
    val = np.where(e == 0, m / 8.0 * 2.0 ** -6, (1.0 + m / 8.0) * np.exp2(e - 7.0))
    val = np.where((e == 15) & (m == 7), np.nan, val)
    return sign * val


def e4m3_encode(v):
    """fp32/fp64 values -> e4m3 bytes: round to nearest, ties to even, saturate to +-448.

    Written from the format definition: pick the binade of |v| (exponent floor(log2|v|),
    clamped below at -6 where the subnormal quantum 2^-9 takes over), divide by that
    binade's quantum 2^(e-3), round half to even, then re-assemble exponent and mantissa
    (a round-up to 8/8 moves into the next binade)."""
    v = np.asarray(v, dtype=np.float64)
    sign = np.signbit(v)
    a = np.abs(v)
    out = np.zeros(v.shape, dtype=np.uint8)
    nan = np.isnan(a)
    a = np.where(nan, 0.0, a)
    with np.errstate(divide="ignore"):
        e = np.floor(np.log2(np.where(a > 0, a, 1.0)))
    e = np.clip(e, -6, 8)
    quantum = np.exp2(e - 3)
    k = np.round(a / quantum)  # numpy rounds half to even
    r = k * quantum  # rounded magnitude, exactly representable
    r = np.minimum(r, E4M3_MAX)  # satfinite
    # re-encode r
    with np.errstate(divide="ignore"):
        er = np.floor(np.log2(np.where(r > 0, r, 1.0)))
    normal = r >= 2.0 ** -6
    exp_field = np.where(normal, er + 7, 0).astype(np.int64)
    mant = np.where(normal, np.round((r / np.exp2(er) - 1.0) * 8), np.round(r / 2.0 ** -9)).astype(np.int64)
    code = (exp_field << 3) | mant
    code = np.where(r == 0, 0, code)
    code = code | np.where(sign, 0x80, 0)
    code = np.where(nan, 0x7F, code)
    out[...] = code.astype(np.uint8)
    return out


def quantize_per_tensor(x):
    """x (fp32-representable, e.g. bf16 values) -> (q bytes, s fp32): R28's current scaling."""
    x32 = np.asarray(x, dtype=np.float32)
    amax = np.float32(np.max(np.abs(x32))) if x32.size else np.float32(0)
    s = np.float32(amax / np.float32(E4M3_MAX)) if amax > 0 else np.float32(1.0)
    y = (x32 / s).astype(np.float32)  # IEEE fp32 division, round to nearest even
    return e4m3_encode(y), s


def gemm_e4m3(qa, qb, sa, sb):
    """out[M, N] = sa * sb * dec(qa)[M, K] . dec(qb)[N, K]^T in fp64."""
    return float(sa) * float(sb) * (e4m3_decode(qa) @ e4m3_decode(qb).T)


# ---------------------------------------------------------------- MXFP8 (R30)
# OCP Microscaling (MX) Formats Specification v1.0, MXFP8 with E4M3 elements: a block of 32
# consecutive elements (along K) shares one E8M0 scale X = 2^e (e + 127 stored in a byte,
# 255 = NaN unused here).  Conversion (spec §6.3): e = floor(log2(max_i |V_i|)) - emax_elem,
# emax_elem = 8 for E4M3 (448 = 1.75 * 2^8), clamped to the E8M0 range [-127, 127]; each
# element P_i = e4m3(V_i / X), rounded to nearest even and clamped to +-448 (so a block whose
# amax mantissa exceeds 1.75 saturates its largest elements -- the spec's behaviour, kept).
# An all-zero block takes e = -127 (byte 0) and zero codes.  The division by the power of two
# X is exact in fp64 (and in the kernel's fp32 unless the quotient falls below 2^-126, where
# every e4m3 code is 0 on both sides).
MX_BLOCK = 32
E4M3_EMAX = 8


def mx_quantize(x):
    """x [R, K] (K % 32 == 0, fp32-representable) -> (q uint8 [R, K], sbytes uint8 [R, K/32])."""
    x = np.asarray(x, dtype=np.float64)
    R, K = x.shape
    assert K % MX_BLOCK == 0
    xb = x.reshape(R, K // MX_BLOCK, MX_BLOCK)
    amax = np.max(np.abs(xb), axis=-1)
    with np.errstate(divide="ignore"):
        e = np.floor(np.log2(np.where(amax > 0, amax, 1.0))) - E4M3_EMAX
    e = np.where(amax > 0, e, -127.0)
    e = np.clip(e, -127, 127)
    q = e4m3_encode(xb / np.exp2(e)[..., None]).reshape(R, K)
    return q, (e + 127).astype(np.uint8)


def mx_dequantize(q, sbytes):
    """(q [R, K], sbytes [R, K/32]) -> fp64 values dec(q) * 2^(s - 127)."""
    q = np.asarray(q, dtype=np.uint8)
    R, K = q.shape
    sc = np.exp2(np.asarray(sbytes, dtype=np.float64) - 127.0)
    return (e4m3_decode(q).reshape(R, K // MX_BLOCK, MX_BLOCK) * sc[..., None]).reshape(R, K)


def gemm_mxf8(qa, sa, qb, sb):
    """out[M, N] = mx_dequantize(qa, sa) . mx_dequantize(qb, sb)^T in fp64 (every product of
    two MXFP8 values is exact in fp64)."""
    return mx_dequantize(qa, sa) @ mx_dequantize(qb, sb).T
