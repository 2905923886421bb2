"""Pins for the oracle's DiT arithmetic against closed forms, brute force and
invariants.  None of these re-types the oracle's formula:
each checks a consequence that a dropped term, wrong sign/index or transposed
operand would break."""
import itertools
import math

import numpy as np
import pytest

from oracle import dit
from oracle import params as OP
from synth.configs import TINY, MID, IMAGE, VIDEO, with_layers


# ---------------------------------------------------------------- P4 schedule
@pytest.mark.parametrize("shift,want", [
    (1.0, [1, .75, .5, .25, 0]),
    (3.0, [1, .9, .75, .5, 0]),
    (5.0, [1, .9375, 5 / 6, .625, 0]),
])
def test_sigma_worked_values(shift, want):
    np.testing.assert_allclose(dit.sigmas(4, shift), want, rtol=0, atol=1e-15)


# ---------------------------------------------------------------- P1-P3 Euler
def _euler_run(field, x0, sig):
    x = x0.copy()
    for i in range(len(sig) - 1):
        x = dit.euler_update(x, field(x, sig[i]), sig[i], sig[i + 1])
    return x


@pytest.mark.parametrize("S,shift", [(4, 1.0), (28, 3.0), (50, 5.0)])
def test_euler_constant_field(S, shift):
    # v == c  =>  x_S = x0 + c * (sigma_S - sigma_0) = x0 - c
    x0 = np.linspace(-1, 1, 7)
    c = np.linspace(0.3, -2, 7)
    xs = _euler_run(lambda x, s: c, x0, dit.sigmas(S, shift))
    np.testing.assert_allclose(xs, x0 - c, atol=1e-14)


@pytest.mark.parametrize("S,shift", [(4, 1.0), (28, 3.0), (50, 5.0)])
def test_euler_linear_field(S, shift):
    a = 0.7
    sig = dit.sigmas(S, shift)
    x0 = np.array([1.0, -2.0, 0.5])
    xs = _euler_run(lambda x, s: a * x, x0, sig)
    np.testing.assert_allclose(xs, np.prod(1 + a * np.diff(sig)) * x0, rtol=1e-14)
    # first-order convergence to exp(-a) x0
    fine = _euler_run(lambda x, s: a * x, x0, dit.sigmas(4000, 1.0))
    np.testing.assert_allclose(fine, math.exp(-a) * x0, rtol=1e-3)


@pytest.mark.parametrize("S,shift", [(4, 1.0), (28, 3.0), (50, 5.0)])
def test_euler_rectified_flow_field_hits_target(S, shift):
    # v(x, s) = (x - xhat)/s  =>  x_S = xhat exactly (sigma_S = 0)
    xhat = np.array([0.25, -1.5, 3.0])
    x0 = np.array([2.0, 0.0, -1.0])
    xs = _euler_run(lambda x, s: (x - xhat) / s, x0, dit.sigmas(S, shift))
    np.testing.assert_allclose(xs, xhat, atol=1e-14)


# ---------------------------------------------------------------- P5 attention
def _loop_attention(q, k, v):
    H, Nq, dh = q.shape
    Nk = k.shape[1]
    o = np.zeros((H, Nq, dh))
    for h in range(H):
        for i in range(Nq):
            logits = [sum(q[h, i, t] * k[h, j, t] for t in range(dh)) / math.sqrt(dh) for j in range(Nk)]
            m = max(logits)
            ws = [math.exp(x - m) for x in logits]
            z = sum(ws)
            for t in range(dh):
                o[h, i, t] = sum(ws[j] * v[h, j, t] for j in range(Nk)) / z
    return o


def test_attention_bruteforce():
    r = np.random.default_rng(0)
    q, k, v = r.normal(size=(2, 5, 4)), r.normal(size=(2, 7, 4)), r.normal(size=(2, 7, 4))
    np.testing.assert_allclose(dit.softmax_attention(q, k, v), _loop_attention(q, k, v), atol=1e-13)


def test_attention_special_cases():
    r = np.random.default_rng(1)
    v = r.normal(size=(3, 6, 8))
    # q = 0 -> equal logits -> mean of V
    o = dit.softmax_attention(np.zeros((3, 4, 8)), r.normal(size=(3, 6, 8)), v)
    np.testing.assert_allclose(o, np.broadcast_to(v.mean(axis=1, keepdims=True), o.shape), atol=1e-14)
    # one key -> V
    v1 = r.normal(size=(3, 1, 8))
    o = dit.softmax_attention(r.normal(size=(3, 4, 8)), r.normal(size=(3, 1, 8)), v1)
    np.testing.assert_allclose(o, np.broadcast_to(v1, o.shape), atol=1e-14)
    # one dominant logit -> that row of V
    k = np.zeros((1, 5, 2))
    k[0, 3] = [100.0, 0]
    o = dit.softmax_attention(np.array([[[10.0, 0]]]), k, r.normal(size=(1, 5, 2)) * 0 + np.arange(10).reshape(1, 5, 2))
    np.testing.assert_allclose(o[0, 0], [6.0, 7.0], atol=1e-12)


# ---------------------------------------------------------------- P6 RoPE
def test_rope_invariants():
    cfg = with_layers(MID, 1)
    r = np.random.default_rng(2)
    N, H, dh = 50, 2, cfg.dh
    pos = np.stack([r.integers(0, 5, N), r.integers(0, 32, N), r.integers(0, 32, N)], axis=1)
    u = r.normal(size=(N, H, dh))
    ru = dit.rope3(u, pos, cfg.rope_axes, cfg.rope_theta)
    # each pair keeps its norm
    np.testing.assert_allclose(ru[..., 0::2] ** 2 + ru[..., 1::2] ** 2, u[..., 0::2] ** 2 + u[..., 1::2] ** 2, rtol=1e-12)
    # origin is the identity
    z = dit.rope3(u[:1], np.zeros((1, 3), int), cfg.rope_axes, cfg.rope_theta)
    np.testing.assert_allclose(z, u[:1], atol=0)
    # <R(p) q, R(p') k> = <q, R(p' - p) k>
    q, k = r.normal(size=(1, 1, dh)), r.normal(size=(1, 1, dh))
    p, p2 = np.array([[3, 7, 11]]), np.array([[1, 20, 4]])
    lhs = np.sum(dit.rope3(q, p, cfg.rope_axes, cfg.rope_theta) * dit.rope3(k, p2, cfg.rope_axes, cfg.rope_theta))
    rhs = np.sum(q * dit.rope3(k, p2 - p, cfg.rope_axes, cfg.rope_theta))
    assert abs(lhs - rhs) < 1e-11
    # f = 0 leaves the first D_f dims unchanged, h/w rotate the rest
    Df = cfg.rope_axes[0]
    z = dit.rope3(u[:1], np.array([[0, 3, 5]]), cfg.rope_axes, cfg.rope_theta)
    np.testing.assert_allclose(z[..., :Df], u[:1, :, :Df], atol=0)
    assert not np.allclose(z[..., Df:], u[:1, :, Df:])
    # axis assignment: only the w-axis block moves when only w changes
    z = dit.rope3(u[:1], np.array([[0, 0, 5]]), cfg.rope_axes, cfg.rope_theta)
    np.testing.assert_allclose(z[..., :Df + cfg.rope_axes[1]], u[:1, :, :Df + cfg.rope_axes[1]], atol=0)
    # pair (2m, 2m+1) at angle phi: first w pair rotates by exactly pos_w (j = 0)
    m = (Df + cfg.rope_axes[1]) // 2
    c, s = math.cos(5.0), math.sin(5.0)
    a, b = u[0, 0, 2 * m], u[0, 0, 2 * m + 1]
    np.testing.assert_allclose(z[0, 0, 2 * m:2 * m + 2], [a * c - b * s, a * s + b * c], rtol=1e-13)


def test_rope_axes_split():
    assert IMAGE.rope_axes == (44, 42, 42) and VIDEO.rope_axes == (44, 42, 42)
    assert TINY.rope_axes == (8, 4, 4)


# ---------------------------------------------------------------- P7 RMSNorm
def test_rmsnorm_invariants():
    r = np.random.default_rng(3)
    x = r.normal(size=(6, 64))
    y = dit.rms_norm(x, 0.0)
    np.testing.assert_allclose(np.sqrt(np.mean(y * y, axis=-1)), 1.0, rtol=1e-14)
    np.testing.assert_allclose(dit.rms_norm(7.5 * x, 0.0), y, rtol=1e-13)
    hn = dit.head_rms_norm(x, 4, 0.0).reshape(6, 4, 16)
    np.testing.assert_allclose(np.sqrt(np.mean(hn * hn, axis=-1)), 1.0, rtol=1e-14)


# ---------------------------------------------------------------- P9 patchify
@pytest.mark.parametrize("cfg", [TINY, MID])
def test_patchify_roundtrip_and_index(cfg):
    x = np.random.default_rng(4).normal(size=cfg.latent_shape)
    X = dit.patchify(x, cfg)
    assert X.shape == (cfg.N, cfg.P)
    np.testing.assert_array_equal(dit.unpatchify(X, cfg), x)
    # hand-indexed element: token (f=0, hh=1, ww=2), channel c=1, (i,j,k) = (0,1,0)
    n = (0 * cfg.Hp + 1) * cfg.Wp + 2
    p = ((1 * cfg.pt + 0) * cfg.ph + 1) * cfg.pw + 0
    assert X[n, p] == x[1, 0, 1 * cfg.ph + 1, 2 * cfg.pw + 0]


def test_token_counts():
    assert TINY.N == 16 and IMAGE.N == 4096 and VIDEO.N == 32760 and MID.N == 1024
    assert IMAGE.P == 64 and VIDEO.ffn == 13824 and IMAGE.ffn == 8192


# ---------------------------------------------------------------- P10 + scalar fns
def test_sinusoid_t0_and_scalars():
    s = dit.sinusoid(0.0, 256)
    np.testing.assert_array_equal(s, np.concatenate([np.ones(128), np.zeros(128)]))
    # last frequency is 10000^(-127/128)
    s = dit.sinusoid(1.0, 256)
    assert abs(s[127] - math.cos(10000 ** (-127 / 128))) < 1e-15
    assert abs(dit.silu(1.0) - 0.7310585786300049) < 1e-15
    assert abs(dit.gelu_tanh(1.0) - 0.8411919906082768) < 1e-12
    assert dit.gelu_tanh(0.0) == 0.0


# ---------------------------------------------------------------- P8 adaLN-zero
def test_adaln_zero_block_is_identity():
    cfg = with_layers(TINY, 1)
    P = OP.Params(cfg, 0)
    r0 = np.random.default_rng(5).normal(size=(cfg.N, cfg.d))
    e6 = np.random.default_rng(6).normal(size=(6, cfg.d)) * 0.1
    mod = P.layer(0, "mod").copy()
    mod[2] = -e6[2]      # g1 = 0
    mod[5] = -e6[5]      # g2 = 0
    P.set("L0.mod", mod)
    P.set("L0.co_w", np.zeros((cfg.d, cfg.d)))
    P.set("L0.co_b", np.zeros(cfg.d))
    kv = (np.ones((cfg.L_txt, cfg.d)), np.ones((cfg.L_txt, cfg.d)))
    r1 = dit.block(P, cfg, 0, r0, e6, kv, dit.token_positions(cfg))
    np.testing.assert_array_equal(r1, r0)
    # and a non-zero gate changes it (the wiring is live)
    P.set("L0.mod", P.layer(0, "mod") + np.eye(6, cfg.d) * 0)
    mod2 = mod.copy(); mod2[2] += 0.1
    P.set("L0.mod", mod2)
    assert not np.array_equal(dit.block(P, cfg, 0, r0, e6, kv, dit.token_positions(cfg)), r0)


def test_cross_attention_uses_text():
    # permuting text tokens leaves cross-attn invariant (set semantics, no mask/positions),
    # while changing one token's K/V changes the output
    cfg = with_layers(TINY, 1)
    P = OP.Params(cfg, 0)
    r0 = np.random.default_rng(7).normal(size=(cfg.N, cfg.d))
    e6 = np.zeros((6, cfg.d))
    rr = np.random.default_rng(8)
    kc, vc = rr.normal(size=(cfg.L_txt, cfg.d)), rr.normal(size=(cfg.L_txt, cfg.d))
    pos = dit.token_positions(cfg)
    a = dit.block(P, cfg, 0, r0, e6, (kc, vc), pos)
    perm = rr.permutation(cfg.L_txt)
    b = dit.block(P, cfg, 0, r0, e6, (kc[perm], vc[perm]), pos)
    np.testing.assert_allclose(a, b, atol=1e-12)
    vc2 = vc.copy(); vc2[0] += 1.0
    c = dit.block(P, cfg, 0, r0, e6, (kc, vc2), pos)
    assert np.abs(c - a).max() > 1e-6


def test_block_rows_matches_block():
    # the row-restricted evaluation is the same definition (pins block_rows to block)
    cfg = with_layers(MID, 1)
    P = OP.Params(cfg, 0)
    rr = np.random.default_rng(9)
    r0 = rr.normal(size=(cfg.N, cfg.d))
    e6 = rr.normal(size=(6, cfg.d)) * 0.1
    kv = (rr.normal(size=(cfg.L_txt, cfg.d)), rr.normal(size=(cfg.L_txt, cfg.d)))
    pos = dit.token_positions(cfg)
    full = dit.block(P, cfg, 0, r0, e6, kv, pos)
    rows = np.array([0, 5, 511, 1023])
    np.testing.assert_allclose(dit.block_rows(P, cfg, 0, r0, e6, kv, pos, rows), full[rows], rtol=1e-12, atol=1e-12)


def test_cfg_guidance_pins():
    # g = 1 -> the conditional velocity; g = 0 -> the unconditional one; v(g) affine in g
    cfg = with_layers(TINY, 2)
    P = OP.Params(cfg, 0)
    r = np.random.default_rng(11)
    sig = dit.sigmas(cfg.steps, cfg.shift)
    c1 = dit.prologue(P, cfg, r.normal(size=(cfg.L_txt, cfg.d_txt)), sig)
    c0 = dit.prologue(P, cfg, r.normal(size=(cfg.L_txt, cfg.d_txt)), sig)
    x = r.normal(size=cfg.latent_shape)
    v1 = dit.velocity(P, cfg, x, 1, c1)
    v0 = dit.velocity(P, cfg, x, 1, c0)
    np.testing.assert_allclose(dit.velocity_cfg(P, cfg, x, 1, c1, c0, 1.0), v1, rtol=0, atol=1e-13)
    np.testing.assert_allclose(dit.velocity_cfg(P, cfg, x, 1, c1, c0, 0.0), v0, rtol=0, atol=1e-13)
    a, b, c = (dit.velocity_cfg(P, cfg, x, 1, c1, c0, g) for g in (2.0, 5.0, 8.0))
    np.testing.assert_allclose(c - b, b - a, atol=1e-11)       # affine in g
    assert np.linalg.norm(v1 - v0) > 1e-3 * np.linalg.norm(v1)  # the negative prompt matters


# ---------------------------------------------------------------- I2V (NEXT-3)
def _i2v_cfg():
    from synth.configs import TINY_I2V
    return with_layers(TINY_I2V, 1)


def test_i2v_patch_input_is_channel_concat():
    # the first P patch features are the noisy latent's, the rest y's (Conv3d order over
    # the C + C_y channels): catches a swapped or interleaved concatenation
    from synth import inputs
    cfg = _i2v_cfg()
    x = np.random.default_rng(21).normal(size=cfg.latent_shape)
    y = inputs.y_cond(cfg, 3).astype(np.float64)
    X = dit.patchify(np.concatenate([x, y], 0), cfg)
    assert X.shape == (cfg.N, cfg.P_in)
    np.testing.assert_array_equal(X[:, :cfg.P], dit.patchify(x, cfg))
    np.testing.assert_array_equal(X[:, cfg.P:], dit.patchify(y, cfg))
    # y's first-frame mask reaches exactly the frame-0 tokens
    ppf = cfg.pt * cfg.ph * cfg.pw
    mask_cols = X[:, cfg.P:cfg.P + 4 * ppf]
    f = dit.token_positions(cfg)[:, 0]
    assert np.all(mask_cols[f == 0] == 1.0) and np.all(mask_cols[f > 0] == 0.0)


def _cross_only_block(P, cfg, r0, e6):
    mod = P.layer(0, "mod").copy()
    mod[2] = -e6[2]  # g1 = 0: no self-attention
    mod[5] = -e6[5]  # g2 = 0: no MLP
    P.set("L0.mod", mod)


def test_i2v_single_image_token_adds_its_value_row():
    # L_img = 1: softmax over one key is 1, so the image term is Vi[0] for every query and
    # the block (self-attention and MLP gated off) moves by exactly Vi[0] W_co on every row
    cfg = _i2v_cfg()
    P = OP.Params(cfg, 0)
    rr = np.random.default_rng(22)
    r0 = rr.normal(size=(cfg.N, cfg.d))
    e6 = rr.normal(size=(6, cfg.d)) * 0.1
    _cross_only_block(P, cfg, r0, e6)
    kv = (rr.normal(size=(cfg.L_txt, cfg.d)), rr.normal(size=(cfg.L_txt, cfg.d)))
    ki, vi = rr.normal(size=(1, cfg.d)), rr.normal(size=(1, cfg.d))
    pos = dit.token_positions(cfg)
    a = dit.block(P, cfg, 0, r0, e6, kv, pos)
    b = dit.block(P, cfg, 0, r0, e6, kv, pos, kvi=(ki, vi))
    want = np.broadcast_to(vi[0] @ P.layer(0, "co_w"), (cfg.N, cfg.d))
    np.testing.assert_allclose(b - a, want, rtol=0, atol=1e-12)


def test_i2v_image_tokens_are_a_set():
    # permuting image tokens leaves the block invariant; changing one token's value does not
    cfg = _i2v_cfg()
    P = OP.Params(cfg, 0)
    rr = np.random.default_rng(23)
    r0 = rr.normal(size=(cfg.N, cfg.d))
    e6 = rr.normal(size=(6, cfg.d)) * 0.1
    kv = (rr.normal(size=(cfg.L_txt, cfg.d)), rr.normal(size=(cfg.L_txt, cfg.d)))
    ki, vi = rr.normal(size=(cfg.L_img, cfg.d)), rr.normal(size=(cfg.L_img, cfg.d))
    pos = dit.token_positions(cfg)
    a = dit.block(P, cfg, 0, r0, e6, kv, pos, kvi=(ki, vi))
    perm = rr.permutation(cfg.L_img)
    b = dit.block(P, cfg, 0, r0, e6, kv, pos, kvi=(ki[perm], vi[perm]))
    np.testing.assert_allclose(a, b, atol=1e-12)
    vi2 = vi.copy(); vi2[1] += 1.0
    assert np.abs(dit.block(P, cfg, 0, r0, e6, kv, pos, kvi=(ki, vi2)) - a).max() > 1e-6


def test_i2v_reduces_to_t2v_when_image_paths_are_zero():
    # zero y's patch weights and the image values: the I2V velocity equals the text-only
    # model's with the same (shared tensor-id) weights -> pins the whole I2V wiring to the
    # T2V path and its own pins
    import dataclasses
    from synth import inputs
    cfg = with_layers(_i2v_cfg(), 2)
    t2v = dataclasses.replace(cfg, C_y=0, L_img=0, d_img=0, name="tiny-i2v-as-t2v")
    P = OP.Params(cfg, 0)
    Pt = OP.Params(t2v, 0)
    pw = P["patch_w"].copy(); pw[cfg.P:] = 0.0
    P.set("patch_w", pw)
    Pt.set("patch_w", pw[:cfg.P])
    for l in range(cfg.layers):
        P.set(f"L{l}.vi_w", np.zeros((cfg.d, cfg.d)))
        P.set(f"L{l}.vi_b", np.zeros(cfg.d))
    sig = dit.sigmas(cfg.steps, cfg.shift)
    ctx = np.random.default_rng(24).normal(size=(cfg.L_txt, cfg.d_txt))
    clip = np.random.default_rng(25).normal(size=(cfg.L_img, cfg.d_img))
    y = inputs.y_cond(cfg, 4).astype(np.float64)
    x = np.random.default_rng(26).normal(size=cfg.latent_shape)
    ci = dit.prologue(P, cfg, ctx, sig, clip=clip, y=y)
    ct = dit.prologue(Pt, t2v, ctx, sig)
    np.testing.assert_allclose(dit.velocity(P, cfg, x, 1, ci), dit.velocity(Pt, t2v, x, 1, ct), rtol=0, atol=1e-12)
    # and with the real weights both conditioning paths matter
    P2 = OP.Params(cfg, 0)
    ci2 = dit.prologue(P2, cfg, ctx, sig, clip=clip, y=y)
    v = dit.velocity(P2, cfg, x, 1, ci2)
    ci3 = dit.prologue(P2, cfg, ctx, sig, clip=clip * 0.0, y=y)
    ci4 = dit.prologue(P2, cfg, ctx, sig, clip=clip, y=y * 0.0)
    assert np.linalg.norm(dit.velocity(P2, cfg, x, 1, ci3) - v) > 1e-3 * np.linalg.norm(v)
    assert np.linalg.norm(dit.velocity(P2, cfg, x, 1, ci4) - v) > 1e-3 * np.linalg.norm(v)
