"""ORACLE (test infrastructure only — see oracle/__init__.py).

The boundary stages and the serial pipeline definition.

The paper's E and D stages are LightX2V's T5/CLIP/VAE encoders and VAE decoder
(P:L252); trained weights are out of scope, so both are
random-init stand-ins whose only job is to produce/consume the handoff
payloads with the paper's shapes (R17):

  E  ids_j = Philox(seed, j; c2=0, c3=2) mod V           (tokens, when not given)
     z = Emb[ids];  a = RMSNorm(z) g_a
     z = z + (SiLU(a W_1e) * (a W_3e)) W_2e
     ctx = bf16_RNE(fp32(RMSNorm(z) g_f))                  (E->T payload, bf16)
  T  x0 ~ N(0,1) from Philox(seed; c3=1), Box-Muller;  x_S = EulerLoop_S(DiT, x0, ctx)
  D  per latent frame phi, pixel (y,x):
     u = SiLU(x[:,phi,y,x] W_d1 + b_d1);  o = tanh(u W_d2^(phi==0 ? f : r) + b)
     pixel shuffle ((ch*r+tau)*8+dy)*8+dx -> out[ch, t(phi,tau), 8y+dy, 8x+dx]

The method is "the serial result, just faster": queues, chunks
and overlap never change a number, so the pipeline oracle is
out = D(EulerLoop_S(DiT, x0(seed), E(tokens))).
"""
from __future__ import annotations

import math

import numpy as np

from . import dit
from .philox import stream_words


def bf16_round(x: np.ndarray) -> np.ndarray:
    """fp64 -> fp32 (RNE) -> bf16 (RNE), returned as fp64 values and bits."""
    from .params import f32_to_bf16_rne_bits, bf16_bits_to_f64
    bits = f32_to_bf16_rne_bits(np.asarray(x, dtype=np.float32))
    return bf16_bits_to_f64(bits), bits


def tokens_from_seed(cfg, seed: int, negative: bool = False) -> np.ndarray:
    """Prompt token ids (stream c3=2) or the negative prompt's (stream c3=4)."""
    return (stream_words(seed, cfg.L_txt, 0, 4 if negative else 2) % np.uint32(cfg.vocab)).astype(np.int32)


def noise(cfg, seed: int) -> np.ndarray:
    """x0[j] = fp32_RNE( sqrt(-2 ln u1) cos(2 pi u2) ), u1 = (a+1) 2^-32, u2 = b 2^-32,
    (a, b) = words (2(j&1), 2(j&1)+1) of Philox block j>>1 of stream (seed; 0, 1)."""
    n = cfg.latent_elems
    w = stream_words(seed, 2 * n + 2, 0, 1)[: 2 * n].reshape(n, 2).astype(np.float64)
    u1 = (w[:, 0] + 1.0) * 2.0 ** -32
    u2 = w[:, 1] * 2.0 ** -32
    z = np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * math.pi * u2)
    return z.astype(np.float32).reshape(cfg.latent_shape)


def image_encoder(cfg, seed: int):
    """I2V E stand-in (NEXT-3, R27): the conditioning image's CLIP tokens and VAE latent.
    No trained encoders exist here (OUT), so both are drawn from the request seed with the
    weights' exact uniform recipe (r = (u >> 8) 2^-24; v = fp32_RNE((2r - 1) * fp32(sqrt 3)),
    unit variance): clip[j] = bf16_RNE(v_j) from stream (seed; 0, 5); y channels 0..3 = the
    first-frame mask (1 on latent frame 0), channels 4.. of frame 0 = v_j from stream
    (seed; 0, 6) in [C_y - 4, H, W] row-major order, later frames 0.
    Returns (clip bf16 bits [L_img, d_img], y fp32 [C_y, F, H, W])."""
    a = np.float32(math.sqrt(3.0))

    def uni(n, c3):
        u = stream_words(seed, n, 0, c3)
        r = (u >> np.uint32(8)).astype(np.float32) * np.float32(2.0 ** -24)
        return ((np.float32(2.0) * r - np.float32(1.0)).astype(np.float32) * a).astype(np.float32)

    from .params import f32_to_bf16_rne_bits
    clip = f32_to_bf16_rne_bits(uni(cfg.L_img * cfg.d_img, 5)).reshape(cfg.L_img, cfg.d_img)
    y = np.zeros(cfg.y_shape, dtype=np.float32)
    y[:4, 0] = 1.0
    y[4:, 0] = uni((cfg.C_y - 4) * cfg.H * cfg.W, 6).reshape(cfg.C_y - 4, cfg.H, cfg.W)
    return clip, y


def encoder(P, cfg, ids: np.ndarray):
    """E stand-in; returns (ctx values fp64, ctx bf16 bits)."""
    eps = cfg.eps
    z = P["E.emb"][np.asarray(ids, dtype=np.int64)]
    a = dit.rms_norm(z, eps) * P["E.g_a"]
    z = z + (dit.silu(a @ P["E.e_w1"]) * (a @ P["E.e_w3"])) @ P["E.e_w2"]
    return bf16_round(dit.rms_norm(z, eps) * P["E.g_f"])


def decoder(P, cfg, x: np.ndarray) -> np.ndarray:
    """D stand-in; x [C,F,H,W] -> fp32-valued fp64 [3, 1+4(F-1), 8H, 8W]."""
    C, F, H, W = cfg.latent_shape
    out = np.zeros(cfg.out_shape, dtype=np.float64)
    for phi in range(F):
        pix = np.asarray(x[:, phi], dtype=np.float64).reshape(C, H * W).T          # [HW, C]
        u = dit.silu(pix @ P["D.d1_w"] + P["D.d1_b"])
        if phi == 0:
            r, o = 1, np.tanh(u @ P["D.d2f_w"] + P["D.d2f_b"])
        else:
            r, o = 4, np.tanh(u @ P["D.d2r_w"] + P["D.d2r_b"])
        o = o.reshape(H, W, 3, r, 8, 8)                                            # (y,x,ch,tau,dy,dx)
        for tau in range(r):
            t = 0 if phi == 0 else 4 * phi - 3 + tau
            # out[ch, t, 8y+dy, 8x+dx] = o[y, x, ch, tau, dy, dx]
            out[:, t] = o[:, :, :, tau].transpose(2, 0, 3, 1, 4).reshape(3, 8 * H, 8 * W)
    return out


def request(P, cfg, seed: int, ids=None, steps=None, shift=None, guidance: float = 1.0):
    """Serial E -> T -> D for one request (the pipeline's exact result).  guidance != 1 adds
    the negative prompt (tokens from stream c3=4) and classifier-free guidance (NEXT-2)."""
    if ids is None:
        ids = tokens_from_seed(cfg, seed)
    ctx, ctx_bits = encoder(P, cfg, ids)
    ctx_neg = None
    if guidance != 1.0:
        ctx_neg, _ = encoder(P, cfg, tokens_from_seed(cfg, seed, negative=True))
    clip = y = clip_bits = None
    if cfg.i2v:  # the image conditioning rides the E->T payload after ctx (NEXT-3)
        clip_bits, y = image_encoder(cfg, seed)
        clip = (clip_bits.astype(np.uint32) << np.uint32(16)).view(np.float32).astype(np.float64)
        y = y.astype(np.float64)
    x0 = noise(cfg, seed)
    xS = dit.trajectory(P, cfg, x0.astype(np.float64), ctx, steps=steps, shift=shift, ctx_neg=ctx_neg,
                        guidance=guidance, clip=clip, y=y)
    lat = xS.astype(np.float32)                      # T->D payload is fp32 (R21)
    return {"ids": ids, "ctx": ctx, "ctx_bits": ctx_bits, "x0": x0, "latent": lat, "clip_bits": clip_bits,
            "out": decoder(P, cfg, lat.astype(np.float64))}
