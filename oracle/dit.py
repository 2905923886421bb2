"""ORACLE (test infrastructure only — see oracle/__init__.py).

Plain fp64 definition of the DiT stage of DisagFusion's pipeline: "runs the
main denoising backbone (e.g., a Transformer network) for iterative diffusion
timesteps and updates the latent representation" (PAPER.md P:L252,
§sec:decentral-pipeline).  The paper gives no DiT equations; the
block below is BASELINE.json north_star's component list (patchified latent,
self-attention, cross-attention to encoder text embeddings, gated MLP, adaLN
timestep modulation, flow-matching Euler update) made concrete with Wan2.x
conventions (Wan2.2 is the paper's video model).  Every reading is
listed in DESIGN.md "Readings" (R1-R16).

Precision: fp64 everywhere; the only quantisation points are the defined ones
(bf16 weights, the bf16 E->T payload, the fp32 latent between stages).

No blocking, fusion or reordering beyond the definitions; matmul is a library
primitive (numpy/BLAS in fp64).
"""
from __future__ import annotations

import math

import numpy as np


# ---------------------------------------------------------------- primitives
def rms_norm(z: np.ndarray, eps: float) -> np.ndarray:
    """RMSNorm(z) = z / sqrt(mean_j z_j^2 + eps) over the last axis (R2)."""
    return z / np.sqrt(np.mean(z * z, axis=-1, keepdims=True) + eps)


def head_rms_norm(z: np.ndarray, heads: int, eps: float) -> np.ndarray:
    """RMSNorm applied separately to each dh-slice of the last axis (R6)."""
    sh = z.shape
    zz = z.reshape(sh[:-1] + (heads, sh[-1] // heads))
    return rms_norm(zz, eps).reshape(sh)


def silu(z):
    return z / (1.0 + np.exp(-z))


def gelu_tanh(z):
    return 0.5 * z * (1.0 + np.tanh(math.sqrt(2.0 / math.pi) * (z + 0.044715 * z ** 3)))


def softmax_attention(q: np.ndarray, k: np.ndarray, v: np.ndarray) -> np.ndarray:
    """o = softmax(q k^T / sqrt(dh)) v per head; q [H,Nq,dh], k,v [H,Nk,dh]; no mask (R8)."""
    dh = q.shape[-1]
    s = np.einsum("hqd,hkd->hqk", q, k) / math.sqrt(dh)
    s = s - s.max(axis=-1, keepdims=True)
    p = np.exp(s)
    p /= p.sum(axis=-1, keepdims=True)
    return np.einsum("hqk,hkd->hqd", p, v)


# ---------------------------------------------------------------- schedule
def sigmas(S: int, shift: float) -> np.ndarray:
    """Shifted flow-matching schedule (R13): s_i = 1 - i/S,
    sigma_i = shift*s_i / (1 + (shift-1)*s_i), i = 0..S; sigma_0 = 1, sigma_S = 0."""
    s = 1.0 - np.arange(S + 1, dtype=np.float64) / S
    return shift * s / (1.0 + (shift - 1.0) * s)


def euler_update(x: np.ndarray, v: np.ndarray, sig_i: float, sig_next: float) -> np.ndarray:
    """Flow-matching Euler step x <- x + (sigma_{i+1} - sigma_i) v (north_star; R13)."""
    return x + (sig_next - sig_i) * v


def sinusoid(t: float, freq_dim: int = 256) -> np.ndarray:
    """[cos(t w_0..t w_{h-1}) | sin(...)], w_k = 10000^(-k/h), h = freq_dim/2 (R5)."""
    h = freq_dim // 2
    w = np.power(10000.0, -np.arange(h, dtype=np.float64) / h)
    return np.concatenate([np.cos(t * w), np.sin(t * w)])


# ---------------------------------------------------------------- geometry
def patchify(x: np.ndarray, cfg) -> np.ndarray:
    """X[n,p] = x[c, f*pt+i, hh*ph+j, ww*pw+k]; n = (f*Hp+hh)*Wp+ww,
    p = ((c*pt+i)*ph+j)*pw+k  (Conv3d flatten order, R11).  The channel count is x's
    (C for the latent, C + C_y for the I2V input concat(x, y))."""
    C, pt, ph, pw = x.shape[0], cfg.pt, cfg.ph, cfg.pw
    Fp, Hp, Wp = cfg.Fp, cfg.Hp, cfg.Wp
    X = np.empty((cfg.N, C * pt * ph * pw), dtype=np.float64)
    for f in range(Fp):
        for hh in range(Hp):
            for ww in range(Wp):
                n = (f * Hp + hh) * Wp + ww
                blk = x[:, f * pt:(f + 1) * pt, hh * ph:(hh + 1) * ph, ww * pw:(ww + 1) * pw]
                X[n] = blk.reshape(C * pt * ph * pw)  # (c, i, j, k) row-major == p order
    return X


def unpatchify(y: np.ndarray, cfg) -> np.ndarray:
    """Exact inverse of patchify."""
    C, pt, ph, pw = cfg.C, cfg.pt, cfg.ph, cfg.pw
    Fp, Hp, Wp = cfg.Fp, cfg.Hp, cfg.Wp
    x = np.empty(cfg.latent_shape, dtype=np.float64)
    for f in range(Fp):
        for hh in range(Hp):
            for ww in range(Wp):
                n = (f * Hp + hh) * Wp + ww
                x[:, f * pt:(f + 1) * pt, hh * ph:(hh + 1) * ph, ww * pw:(ww + 1) * pw] = \
                    y[n].reshape(C, pt, ph, pw)
    return x


def token_positions(cfg) -> np.ndarray:
    """(f, h, w) grid coordinate of token n (0-based, after patchify)."""
    n = np.arange(cfg.N)
    w = n % cfg.Wp
    h = (n // cfg.Wp) % cfg.Hp
    f = n // (cfg.Wp * cfg.Hp)
    return np.stack([f, h, w], axis=1)


def rope3(u: np.ndarray, pos: np.ndarray, axes, theta: float) -> np.ndarray:
    """3-axis RoPE on head vectors u [N, H, dh] (R7).

    Pair m = (u_{2m}, u_{2m+1}); the first D_f/2 pairs rotate with the f
    coordinate, the next D_h/2 with h, the last D_w/2 with w; within axis a,
    local pair j has angle phi = pos_a * theta^(-2j/D_a).
    u'_{2m} = u_{2m} cos phi - u_{2m+1} sin phi;  u'_{2m+1} = u_{2m} sin phi + u_{2m+1} cos phi.
    """
    N, H, dh = u.shape
    phi = np.empty((N, dh // 2), dtype=np.float64)
    m0 = 0
    for a, Da in enumerate(axes):
        j = np.arange(Da // 2, dtype=np.float64)
        inv = np.power(theta, -2.0 * j / Da)
        phi[:, m0:m0 + Da // 2] = pos[:, a:a + 1].astype(np.float64) * inv[None, :]
        m0 += Da // 2
    c = np.cos(phi)[:, None, :]
    s = np.sin(phi)[:, None, :]
    ue, uo = u[..., 0::2], u[..., 1::2]
    out = np.empty_like(u)
    out[..., 0::2] = ue * c - uo * s
    out[..., 1::2] = ue * s + uo * c
    return out


# ---------------------------------------------------------------- conditioning
def time_embedding(P, cfg, sigma: float):
    """e = SiLU(s W_e1 + b_e1) W_e2 + b_e2 with s = sinusoid(1000 sigma);
    e6 = reshape(SiLU(e) W_m + b_m, [6, d])  (R4, R5)."""
    s = sinusoid(1000.0 * sigma, cfg.freq_dim)
    e = silu(s @ P["temb1_w"] + P["temb1_b"]) @ P["temb2_w"] + P["temb2_b"]
    e6 = (silu(e) @ P["tmod_w"] + P["tmod_b"]).reshape(6, cfg.d)
    return e, e6


def text_projection(P, cfg, ctx: np.ndarray) -> np.ndarray:
    """ctx' = GELU_tanh(ctx W_t1 + b_t1) W_t2 + b_t2  -> [L_txt, d]."""
    return gelu_tanh(ctx @ P["txt1_w"] + P["txt1_b"]) @ P["txt2_w"] + P["txt2_b"]


def cross_kv(P, cfg, l: int, ctxp: np.ndarray):
    """K_l = headRMS(ctx' W_ck + b_ck) * g_ck;  V_l = ctx' W_cv + b_cv  (R3, R6)."""
    k = head_rms_norm(ctxp @ P.layer(l, "ck_w") + P.layer(l, "ck_b"), cfg.heads, cfg.eps) * P.layer(l, "g_ck")
    v = ctxp @ P.layer(l, "cv_w") + P.layer(l, "cv_b")
    return k, v


def image_projection(P, cfg, clip: np.ndarray) -> np.ndarray:
    """I2V (NEXT-3, reading R27): img' = GELU_tanh(clip W_i1 + b_i1) W_i2 + b_i2 -> [L_img, d]
    (the text projection's form; Wan's MLPProj adds LayerNorms)."""
    return gelu_tanh(clip @ P["img1_w"] + P["img1_b"]) @ P["img2_w"] + P["img2_b"]


def image_kv(P, cfg, l: int, imgp: np.ndarray):
    """Ki_l = headRMS(img' W_ki + b_ki) * g_ki;  Vi_l = img' W_vi + b_vi  (as cross_kv)."""
    k = head_rms_norm(imgp @ P.layer(l, "ki_w") + P.layer(l, "ki_b"), cfg.heads, cfg.eps) * P.layer(l, "g_ki")
    v = imgp @ P.layer(l, "vi_w") + P.layer(l, "vi_b")
    return k, v


def prologue(P, cfg, ctx: np.ndarray, sig: np.ndarray, clip=None, y=None):
    """Per-request conditioning: cross K/V for every layer and
    (e_i, e6_i) for every step i < S.  I2V (cfg.C_y > 0): also the image-token K/V of
    every layer from clip [L_img, d_img], and y [C_y, F, H, W] for the patch embedding."""
    ctxp = text_projection(P, cfg, ctx)
    kv = [cross_kv(P, cfg, l, ctxp) for l in range(cfg.layers)]
    te = [time_embedding(P, cfg, float(sig[i])) for i in range(len(sig) - 1)]
    cond = {"ctxp": ctxp, "kv": kv, "e": [t[0] for t in te], "e6": [t[1] for t in te], "kvi": None, "y": None}
    if cfg.i2v:
        imgp = image_projection(P, cfg, np.asarray(clip, dtype=np.float64))
        cond["kvi"] = [image_kv(P, cfg, l, imgp) for l in range(cfg.layers)]
        cond["y"] = np.asarray(y, dtype=np.float64)
    return cond


def _heads(z: np.ndarray, H: int) -> np.ndarray:
    """[N, H*dh] -> [H, N, dh]."""
    N = z.shape[0]
    return z.reshape(N, H, -1).transpose(1, 0, 2)


def _unheads(z: np.ndarray) -> np.ndarray:
    H, N, dh = z.shape
    return z.transpose(1, 0, 2).reshape(N, H * dh)


# ---------------------------------------------------------------- one block
def block(P, cfg, l: int, r: np.ndarray, e6: np.ndarray, kv, pos, cross: bool = True, kvi=None,
          q8=None) -> np.ndarray:
    """One DiT block (Wan2.1 order, R1): adaLN self-attention, cross-attention,
    adaLN gated MLP.  r [N, d] fp64 -> r' [N, d].  I2V: the cross-attention output is the
    text term plus the image-token term softmax(qc Ki^T / sqrt(dh)) Vi (Wan I2V, R27).
    q8 (FP8 step mode, R29; oracle/dit_fp8.py): every GEMM of the block takes q8.act(input)
    and q8.weight(...) instead of its input and weight."""
    d, H, eps = cfg.d, cfg.heads, cfg.eps
    act = (lambda x: x) if q8 is None else q8.act
    wgt = (lambda l_, name: P.layer(l_, name)) if q8 is None else (lambda l_, name: q8.weight(P, l_, name))
    sh1, sc1, g1, sh2, sc2, g2 = (e6 + P.layer(l, "mod"))  # rows 0..5 (R4)
    # --- self-attention (a4-a7)
    h = rms_norm(r, eps) * (1.0 + sc1) + sh1
    qkv = act(h) @ wgt(l, "qkv_w") + P.layer(l, "qkv_b")
    q, k, v = qkv[:, :d], qkv[:, d:2 * d], qkv[:, 2 * d:]
    q = head_rms_norm(q, H, eps) * P.layer(l, "g_q")
    k = head_rms_norm(k, H, eps) * P.layer(l, "g_k")
    q = rope3(q.reshape(-1, H, cfg.dh), pos, cfg.rope_axes, cfg.rope_theta)
    k = rope3(k.reshape(-1, H, cfg.dh), pos, cfg.rope_axes, cfg.rope_theta)
    if q8 is not None and hasattr(q8, "qk"):  # FP8 modes (R32): e4m3 Q, K for QK^T
        q, k = q8.qk(P, l, q, "g_q"), q8.qk(P, l, k, "g_k")
    if q8 is not None and hasattr(q8, "vq"):  # FP8 modes (R33): e4m3 V for PV
        v = q8.vq(v)
    o = softmax_attention(q.transpose(1, 0, 2), k.transpose(1, 0, 2), _heads(v, H))
    r = r + g1 * (act(_unheads(o)) @ wgt(l, "o_w") + P.layer(l, "o_b"))
    # --- cross-attention (a8): pre-norm with gain, not modulated, ungated (R3)
    if cross:
        hc = rms_norm(r, eps) * P.layer(l, "g_n3")
        qc = head_rms_norm(act(hc) @ wgt(l, "cq_w") + P.layer(l, "cq_b"), H, eps) * P.layer(l, "g_cq")
        kc, vc = kv
        oc = softmax_attention(_heads(qc, H), _heads(kc, H), _heads(vc, H))
        if kvi is not None:
            oc = oc + softmax_attention(_heads(qc, H), _heads(kvi[0], H), _heads(kvi[1], H))
        r = r + (act(_unheads(oc)) @ wgt(l, "co_w") + P.layer(l, "co_b"))
    # --- gated MLP (a9-a10): SwiGLU with biases (R9)
    h2 = act(rms_norm(r, eps) * (1.0 + sc2) + sh2)
    a = silu(h2 @ wgt(l, "w1") + P.layer(l, "b1")) * (h2 @ wgt(l, "w3") + P.layer(l, "b3"))
    r = r + g2 * (act(a) @ wgt(l, "w2") + P.layer(l, "b2"))
    return r


def block_rows(P, cfg, l: int, r: np.ndarray, e6: np.ndarray, kv, pos, rows, kvi=None) -> np.ndarray:
    """block() evaluated only at output rows `rows` (production-shape parity).
    Same definition: self-attention keys/values use ALL tokens; every other
    operation is row-wise, so restricting the query rows changes nothing."""
    d, H, eps = cfg.d, cfg.heads, cfg.eps
    rows = np.asarray(rows)
    sh1, sc1, g1, sh2, sc2, g2 = (e6 + P.layer(l, "mod"))
    h = rms_norm(r, eps) * (1.0 + sc1) + sh1                        # all rows (K, V need them)
    W = P.layer(l, "qkv_w")
    b = P.layer(l, "qkv_b")
    k = head_rms_norm(h @ W[:, d:2 * d] + b[d:2 * d], H, eps) * P.layer(l, "g_k")
    v = h @ W[:, 2 * d:] + b[2 * d:]
    q = head_rms_norm(h[rows] @ W[:, :d] + b[:d], H, eps) * P.layer(l, "g_q")
    q = rope3(q.reshape(-1, H, cfg.dh), pos[rows], cfg.rope_axes, cfg.rope_theta)
    k = rope3(k.reshape(-1, H, cfg.dh), pos, cfg.rope_axes, cfg.rope_theta)
    o = softmax_attention(q.transpose(1, 0, 2), k.transpose(1, 0, 2), _heads(v, H))
    rr = r[rows] + g1 * (_unheads(o) @ P.layer(l, "o_w") + P.layer(l, "o_b"))
    hc = rms_norm(rr, eps) * P.layer(l, "g_n3")
    qc = head_rms_norm(hc @ P.layer(l, "cq_w") + P.layer(l, "cq_b"), H, eps) * P.layer(l, "g_cq")
    kc, vc = kv
    oc = softmax_attention(_heads(qc, H), _heads(kc, H), _heads(vc, H))
    if kvi is not None:
        oc = oc + softmax_attention(_heads(qc, H), _heads(kvi[0], H), _heads(kvi[1], H))
    rr = rr + (_unheads(oc) @ P.layer(l, "co_w") + P.layer(l, "co_b"))
    h2 = rms_norm(rr, eps) * (1.0 + sc2) + sh2
    a = silu(h2 @ P.layer(l, "w1") + P.layer(l, "b1")) * (h2 @ P.layer(l, "w3") + P.layer(l, "b3"))
    return rr + g2 * (a @ P.layer(l, "w2") + P.layer(l, "b2"))


def head(P, cfg, r: np.ndarray, e: np.ndarray) -> np.ndarray:
    """(sh, sc) = head_mod + e (e un-projected, R12);
    y = (RMSNorm(r)(1+sc)+sh) W_h + b_h;  v = unpatchify(y)."""
    sh, sc = P["head_mod"] + e
    y = (rms_norm(r, cfg.eps) * (1.0 + sc) + sh) @ P["head_w"] + P["head_b"]
    return unpatchify(y, cfg)


def velocity(P, cfg, x: np.ndarray, i: int, cond, cross: bool = True, trace=None, q8=None) -> np.ndarray:
    """v(x_i, sigma_i): patch embed -> blocks -> head (a2-a11)."""
    pos = token_positions(cfg)
    xin = np.asarray(x, dtype=np.float64)
    if cfg.i2v:  # concat(x, y) along channels before patchify (Wan I2V in_dim = C + C_y)
        xin = np.concatenate([xin, cond["y"]], axis=0)
    r = patchify(xin, cfg) @ P["patch_w"] + P["patch_b"]
    if trace is not None:
        trace.append(r.copy())
    kvi = cond.get("kvi")
    for l in range(cfg.layers):
        r = block(P, cfg, l, r, cond["e6"][i], cond["kv"][l], pos, cross=cross,
                  kvi=kvi[l] if kvi is not None else None, q8=q8)
        if trace is not None:
            trace.append(r.copy())
    return head(P, cfg, r, cond["e"][i])


def velocity_cfg(P, cfg, x, i, cond, cond_neg, guidance: float) -> np.ndarray:
    """Classifier-free guidance (NEXT-2; "negative prompts"): the DiT runs on the
    conditional and the negative-prompt conditioning; v = v_u + g (v_c - v_u).  g = 1 is the
    conditional velocity (R20)."""
    v_c = velocity(P, cfg, x, i, cond)
    v_u = velocity(P, cfg, x, i, cond_neg)
    return v_u + guidance * (v_c - v_u)


def step(P, cfg, x, i, cond, sig, q8=None):
    """One denoising step: returns (x_{i+1}, v_i)."""
    v = velocity(P, cfg, x, i, cond, q8=q8)
    return euler_update(np.asarray(x, dtype=np.float64), v, sig[i], sig[i + 1]), v


def trajectory(P, cfg, x0, ctx, steps=None, shift=None, ctx_neg=None, guidance: float = 1.0, clip=None, y=None):
    """x_S from x_0 and the bf16 ctx payload (values as fp64); with ctx_neg, classifier-free
    guidance with scale `guidance`; I2V configs also take clip and y."""
    S = cfg.steps if steps is None else steps
    sig = sigmas(S, cfg.shift if shift is None else shift)
    cond = prologue(P, cfg, ctx, sig, clip=clip, y=y)
    cond_neg = prologue(P, cfg, ctx_neg, sig, clip=clip, y=y) if ctx_neg is not None else None
    x = np.asarray(x0, dtype=np.float64)
    for i in range(S):
        if cond_neg is None:
            x, _ = step(P, cfg, x, i, cond, sig)
        else:
            x = euler_update(x, velocity_cfg(P, cfg, x, i, cond, cond_neg, guidance), sig[i], sig[i + 1])
    return x
