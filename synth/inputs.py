"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

Holds none of the method's arithmetic: every function here only draws random
numbers (numpy PCG64, seeded) with the shapes and value distributions of the
paper's workloads.  The method's own random draws
(weights, noise x0, token ids) are NOT made here: each side implements the
same counter-based Philox4x32-10 generator independently.
"""
from __future__ import annotations

import numpy as np


def rng(seed: int) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence([0xD15A6F05, int(seed)]))


def f32_to_bf16_bits_trunc(a: np.ndarray) -> np.ndarray:
    """Input generation only: take the top 16 bits of an fp32 (a bf16 value by
    construction, no rounding decision involved)."""
    return (np.ascontiguousarray(a, dtype=np.float32).view(np.uint32) >> 16).astype(np.uint16)


def bf16_bits_to_f64(b: np.ndarray) -> np.ndarray:
    return (b.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def latent(cfg, seed: int) -> np.ndarray:
    """A latent x_i of shape [C,F,H,W] fp32, N(0,1) (the flow-matching prior)."""
    return rng(seed).standard_normal(cfg.latent_shape, dtype=np.float32)


def ctx_bf16(cfg, seed: int) -> np.ndarray:
    """An encoder output (E->T payload) [L_txt, d_txt] as bf16 bits, values ~N(0,1)
    like an RMS-normalised hidden state."""
    return f32_to_bf16_bits_trunc(rng(seed).standard_normal((cfg.L_txt, cfg.d_txt), dtype=np.float32))


def clip_bf16(cfg, seed: int) -> np.ndarray:
    """I2V image tokens (E->T payload) [L_img, d_img] as bf16 bits, values ~N(0,1)."""
    return f32_to_bf16_bits_trunc(rng(seed).standard_normal((cfg.L_img, cfg.d_img), dtype=np.float32))


def y_cond(cfg, seed: int) -> np.ndarray:
    """I2V conditioning y [C_y, F, H, W] fp32 (Wan layout): channels 0..3 the first-frame
    mask (1 on latent frame 0, 0 elsewhere), channels 4.. a VAE-like latent of the conditioning
    image on frame 0 (N(0,1)) and zeros on the later frames."""
    y = np.zeros(cfg.y_shape, dtype=np.float32)
    y[:4, 0] = 1.0
    y[4:, 0] = rng(seed).standard_normal((cfg.C_y - 4, cfg.H, cfg.W), dtype=np.float32)
    return y


def residual(cfg, seed: int, scale: float = 1.0) -> np.ndarray:
    """A DiT residual stream r [N, d] fp32 (input of one block)."""
    return (scale * rng(seed).standard_normal((cfg.N, cfg.d), dtype=np.float32)).astype(np.float32)


def token_ids(cfg, seed: int) -> np.ndarray:
    return rng(seed).integers(0, cfg.vocab, size=cfg.L_txt, dtype=np.int32)


def int_matrix(shape, lo: int, hi: int, seed: int) -> np.ndarray:
    """Integer-valued matrix (for bit-exact GEMM pins), as fp32."""
    return rng(seed).integers(lo, hi + 1, size=shape).astype(np.float32)


def payload_bytes(nbytes: int, seed: int) -> np.ndarray:
    return rng(seed).integers(0, 256, size=nbytes, dtype=np.uint8)


def activation_bf16(shape, seed: int, outlier_frac: float = 1e-3, outlier_scale: float = 24.0) -> np.ndarray:
    """bf16 bits of an activation-like matrix: N(0,1) with a sparse set of large-magnitude
    outliers (the channel outliers that make per-tensor FP8 scaling lossy, NEXT-4)."""
    g = rng(seed)
    a = g.standard_normal(shape, dtype=np.float32)
    m = g.random(shape) < outlier_frac
    a[m] *= np.float32(outlier_scale)
    return f32_to_bf16_bits_trunc(a)
