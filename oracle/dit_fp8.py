"""fp64 CPU ORACLE of the FP8 step mode (R29).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): never imported by the product path.

PAPER.md names quantisation only as a serving optimisation of the systems it builds on
("FP8/INT8 quantisation") and fixes no format.  Reading R29 (on top of R28's E4M3
format and per-tensor current scaling, oracle/fp8.py):
  * all six GEMMs of a block -- QKV (a5), O (a7), cross-Q and cross-O (a8), MLP up W1 | W3
    and MLP down (a10) -- take e4m3 operands; every other operation (norms, attention, the
    prologue, patch embedding, head) is the bf16 model's (oracle/dit.py);
  * a GEMM's input activation x [N, K] is quantised per token row: x is rounded to fp32 (the
    kernel's precision, which decides the codes), s_m = the smallest power of two >=
    fp32(amax_j |x_mj| / 448) (1 for a zero row; a power of two makes x / s_m an exact exponent
    shift), q_mj = e4m3(x_mj / s_m), and the GEMM sees dec(q_mj) * s_m;
  * the weight is quantised per tensor (R28) -- the fused W_qkv as one tensor, W_1 and W_3
    jointly (the GPU stores them interleaved as one tensor) -- and the GEMM sees dec(q) * s;
  * products are exact and summed in fp64 (the GPU: exact products, fp32 accumulation);
  * R32: the self-attention's QK^T also takes e4m3 Q and K (per-layer power-of-two scales from
    the qk-norm gains, qk_scale / qk_quant); R33: its PV takes e4m3 V (per-tensor power-of-two
    scale, v_quant) -- and, on the GPU only, e4m3 P (not mirrored, see v_quant).

Pinned by tests/test_oracle_fp8.py: quantize_rows' closed forms (a row whose amax is 448
keeps its e4m3-representable values; a zero row; power-of-two row scaling moves only the
scale), and the wiring -- block(..., q8=Q8 with identity quantisers) is dit.block exactly,
so the FP8 mode differs from the pinned bf16 composition only where R29 says.  The MXFP8 mode
(R31, below) reuses the same wiring with R30's block quantisers; mx_weight is pinned by its
orientation (scaling one output column by 2^k scales only that column's dequantised weight,
which neither per-tensor scaling nor blocks along N would do) and mx_act by the MX closed forms
of oracle/fp8.py.
"""
from __future__ import annotations

import numpy as np

from . import fp8
from . import dit

E4M3_MAX = np.float32(448.0)


def pow2_ceil(v):
    """Smallest power of two >= v (v > 0, fp32): v itself if it is one."""
    m, e = np.frexp(np.asarray(v, dtype=np.float64))  # v = m 2^e, m in [0.5, 1)
    return np.where(m == 0.5, v, np.ldexp(1.0, e)).astype(np.float32)


def quantize_rows(h):
    """h [M, K] -> (q bytes [M, K], s fp32 [M]): per-row scaling with power-of-two scales (R29)."""
    h32 = np.asarray(h, dtype=np.float64).astype(np.float32)
    amax = np.max(np.abs(h32), axis=-1).astype(np.float32)
    s = np.where(amax > 0, pow2_ceil((amax / E4M3_MAX).astype(np.float32)), np.float32(1.0)).astype(np.float32)
    y = (h32.astype(np.float64) / s.astype(np.float64)[:, None])  # exact: s is a power of two
    return fp8.e4m3_encode(y), s


def act(h):
    """The activation as the e4m3 GEMM sees it: dec(q) * s per row."""
    q, s = quantize_rows(h)
    return fp8.e4m3_decode(q) * s.astype(np.float64)[:, None]


def weight_q(W):
    """The weight as the e4m3 GEMM sees it: dec(q) * s per tensor (R28)."""
    q, s = fp8.quantize_per_tensor(np.asarray(W, dtype=np.float64))
    return fp8.e4m3_decode(q) * float(s)


def qk_scale(g, dh):
    """R32: the power-of-two e4m3 scale of the self-attention's Q (or K) of a layer.  After the
    per-head RMSNorm every head vector has norm sqrt(dh), so after the gain g and the RoPE
    rotation (which keeps each pair's norm) every component is at most sqrt(dh) * max|g|;
    s = the smallest power of two >= fp32(sqrt(dh) * max|g| / 448) keeps every code unsaturated."""
    gmax = float(np.max(np.abs(np.asarray(g, dtype=np.float64))))
    return pow2_ceil(np.float32(np.sqrt(float(dh)) * gmax / 448.0)) if gmax > 0 else np.float32(1.0)


def qk_quant(x, s):
    """Q or K [.., dh] as the e4m3 QK^T sees it: the GPU quantises the bf16 Q / K it stored, so
    x is rounded to bf16 first; dec(e4m3(bf16(x) / s)) * s (the division is exact)."""
    from .stages import bf16_round
    xb, _ = bf16_round(x)
    return fp8.e4m3_decode(fp8.e4m3_encode(xb / float(s))) * float(s)


def v_quant(v):
    """R33: V (all heads of a sample) as the e4m3 PV sees it: the GPU quantises its bf16 V per
    tensor with s = the smallest power of two >= fp32(amax|V| / 448); dec(e4m3(bf16(v) / s)) * s.
    (P's e4m3 rounding inside the kernel depends on its running row maximum and is not
    mirrored: the tolerance covers it, R33.)"""
    from .stages import bf16_round
    vb, _ = bf16_round(v)
    amax = np.float32(np.max(np.abs(vb))) if vb.size else np.float32(0)
    s = pow2_ceil(np.float32(amax / E4M3_MAX)) if amax > 0 else np.float32(1.0)
    return fp8.e4m3_decode(fp8.e4m3_encode(vb / float(s))) * float(s)


class Q8:
    """Quantisers handed to oracle.dit.block (q8=...).  W_1 and W_3 share one scale (they are
    one interleaved tensor on the GPU); the dequantised weights are cached per layer.  qk_fn
    (R32) quantises the self-attention's Q and K with the layer's qk_scale."""

    def __init__(self, act_fn=act, weight_fn=weight_q, qk_fn=qk_quant, v_fn=v_quant):
        self.act = act_fn
        self._wq = weight_fn
        self._qk = qk_fn
        self.vq = v_fn
        self._cache = {}

    def qk(self, P, l, x, gname):
        return self._qk(x, qk_scale(P.layer(l, gname), x.shape[-1]))

    def weight(self, P, l, name):
        key = (id(P), l, name)
        if key not in self._cache:
            if name in ("w1", "w3"):
                w1, w3 = P.layer(l, "w1"), P.layer(l, "w3")
                both = self._wq(np.concatenate([w1, w3], axis=1))
                f = w1.shape[1]
                self._cache[(id(P), l, "w1")] = both[:, :f]
                self._cache[(id(P), l, "w3")] = both[:, f:]
            else:
                self._cache[key] = self._wq(P.layer(l, name))
        return self._cache[key]


def step(P, cfg, x, i, cond, sig):
    """One FP8-mode denoising step: (x_{i+1}, v_i)."""
    return dit.step(P, cfg, x, i, cond, sig, q8=Q8())


# ---------------------------------------------------------------- MXFP8 step mode (R31)
# Same six GEMMs as R29, with R30's MXFP8 (OCP MX, E4M3 elements, one E8M0 scale per 32
# consecutive k) on both operands instead of per-row / per-tensor scaling: the activation is
# rounded to fp32 (the kernel quantises the fp32 RMSNorm output, or the bf16 attention / SwiGLU
# output, which is exact in fp32) and block-quantised along K; a weight W [K, N] is
# block-quantised along K per output column (the GPU quantises W^T [N, K] row by row).
def mx_act(h):
    """The activation as the MXFP8 GEMM sees it."""
    h32 = np.asarray(h, dtype=np.float64).astype(np.float32).astype(np.float64)
    q, s = fp8.mx_quantize(h32)
    return fp8.mx_dequantize(q, s)


def mx_weight(W):
    """W [K, N] as the MXFP8 GEMM sees it (blocks along K of each output column)."""
    q, s = fp8.mx_quantize(np.asarray(W, dtype=np.float64).T)
    return fp8.mx_dequantize(q, s).T


def Q8MX():
    return Q8(act_fn=mx_act, weight_fn=mx_weight)


def step_mx(P, cfg, x, i, cond, sig):
    """One MXFP8-mode denoising step: (x_{i+1}, v_i)."""
    return dit.step(P, cfg, x, i, cond, sig, q8=Q8MX())
