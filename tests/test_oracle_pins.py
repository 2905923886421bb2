"""Pins for the oracle functions the round-1 verdict found unpinned (SURVEY §8(c).5,
DESIGN.md §11): the time embedding, the text projection, cross K/V, the head, the
SwiGLU branch, the modulation rows of the block, the velocity's wiring of e, and the
encoder stand-in.

Each test picks parameters that reduce the function to a value computable BY HAND
(one-hot / identity-like weights, alternating-sign rows whose RMS norm is known,
zero projections that make softmax uniform), so that a plausible misreading --
SiLU on the wrong side, shift and scale swapped, a (d,6) reshape, the norm on V
instead of K, sigma instead of 1000 sigma, a dropped bias or gate -- changes the
number.  `tools/mutate_oracle.py` applies such one-line mutations to a copy of
oracle/ and checks that every one of them fails a pin (log:
profiles/r02_oracle_mutations.txt).  Expected values use only math/numpy scalar
arithmetic, never the oracle function under test.
"""
import math

import numpy as np

from oracle import dit, stages
from oracle import params as OP
from synth.configs import TINY, with_layers

EPS = TINY.eps


def _silu(x):
    return x / (1.0 + math.exp(-x))


def _gelu_tanh(x):
    return 0.5 * x * (1.0 + math.tanh(math.sqrt(2.0 / math.pi) * (x + 0.044715 * x ** 3)))


def _eye(n_in, n_out, scale=1.0):
    w = np.zeros((n_in, n_out))
    k = min(n_in, n_out)
    w[np.arange(k), np.arange(k)] = scale
    return w


def _alt(d):
    """[1, -1, 1, -1, ...]: every element has |x| = 1, so RMSNorm(a * alt) = a/sqrt(a^2+eps) alt."""
    return np.where(np.arange(d) % 2 == 0, 1.0, -1.0)


# ---------------------------------------------------------------- time embedding (R4, R5)
def test_time_embedding_closed_form():
    """W_e1 reads cos(t w_j) + 0.5 sin(t w_j) into column j, W_e2 = 2 I, W_m maps SiLU(e_j)
    to row k of e6 with weight k+1: every output is a scalar formula in t = 1000 sigma."""
    cfg, d, h = TINY, TINY.d, TINY.freq_dim // 2
    P = OP.Params(cfg, 0)
    w1 = np.zeros((cfg.freq_dim, d))
    w1[np.arange(d), np.arange(d)] = 1.0
    w1[h + np.arange(d), np.arange(d)] = 0.5
    b1 = np.linspace(-2.0, 1.0, d)
    b2 = np.linspace(0.0, 0.3, d)
    wm = np.zeros((d, 6 * d))
    bm = np.zeros(6 * d)
    for k in range(6):
        wm[np.arange(d), k * d + np.arange(d)] = k + 1
        bm[k * d:(k + 1) * d] = 0.01 * k
    P.set("temb1_w", w1); P.set("temb1_b", b1)
    P.set("temb2_w", _eye(d, d, 2.0)); P.set("temb2_b", b2)
    P.set("tmod_w", wm); P.set("tmod_b", bm)
    sigma = 0.37
    e, e6 = dit.time_embedding(P, cfg, sigma)
    t = 1000.0 * sigma
    for j in range(d):
        wj = 10000.0 ** (-j / h)
        pre = math.cos(t * wj) + 0.5 * math.sin(t * wj) + b1[j]
        ej = 2.0 * _silu(pre) + b2[j]
        assert abs(e[j] - ej) < 1e-12, (j, e[j], ej)
        for k in range(6):
            assert abs(e6[k, j] - ((k + 1) * _silu(ej) + 0.01 * k)) < 1e-12, (k, j)
    # sigma = 0: the sinusoid is [1 x 128, 0 x 128] (P10) -> pre = 1 + b1
    e0, _ = dit.time_embedding(P, cfg, 0.0)
    np.testing.assert_allclose(e0, [2.0 * _silu(1.0 + b1[j]) + b2[j] for j in range(d)], rtol=0, atol=1e-12)


# ---------------------------------------------------------------- text projection (a1)
def test_text_projection_closed_form():
    """W_t1 = one-hot (d_txt -> first d_txt columns), b_t1 = 0.25 inside the GELU, W_t2 a
    column shift by one with weight 2: ctx'[:, m] = 2 GELU_tanh(ctx[:, m-1] + 0.25) + b2[m]."""
    cfg = TINY
    P = OP.Params(cfg, 0)
    dt, d = cfg.d_txt, cfg.d
    w2 = np.zeros((d, d))
    w2[np.arange(d), (np.arange(d) + 1) % d] = 2.0
    b2 = np.linspace(-0.1, 0.1, d)
    P.set("txt1_w", _eye(dt, d)); P.set("txt1_b", np.full(d, 0.25))
    P.set("txt2_w", w2); P.set("txt2_b", b2)
    ctx = np.random.default_rng(3).normal(size=(cfg.L_txt, dt))
    out = dit.text_projection(P, cfg, ctx)
    for i in range(cfg.L_txt):
        for m in range(d):
            src = (m - 1) % d
            x = ctx[i, src] if src < dt else 0.0
            assert abs(out[i, m] - (2.0 * _gelu_tanh(x + 0.25) + b2[m])) < 1e-12, (i, m)


# ---------------------------------------------------------------- cross K/V (R3, R6)
def test_cross_kv_norms_k_per_head_not_v():
    """K = headRMS(ctx' W_ck + b) g_ck: every head of every row has RMS |g| whatever the
    per-head input scale, and points along its input; V = ctx' W_cv + b_cv un-normalised."""
    cfg = with_layers(TINY, 1)
    P = OP.Params(cfg, 0)
    d, H, dh = cfg.d, cfg.heads, cfg.dh
    scale = np.repeat(np.arange(1, H + 1, dtype=np.float64) * 3.0, dh)      # head h scaled by 3(h+1)
    P.set("L0.ck_w", np.diag(scale)); P.set("L0.ck_b", np.zeros(d))
    P.set("L0.g_ck", np.full(d, 1.5))
    bv = np.linspace(-1, 1, d)
    P.set("L0.cv_w", _eye(d, d, 3.0)); P.set("L0.cv_b", bv)
    ctxp = np.random.default_rng(4).normal(size=(cfg.L_txt, d))
    k, v = dit.cross_kv(P, cfg, 0, ctxp)
    np.testing.assert_allclose(v, 3.0 * ctxp + bv, rtol=0, atol=1e-12)
    for i in range(cfg.L_txt):
        for hh in range(H):
            kh, uh = k[i, hh * dh:(hh + 1) * dh], ctxp[i, hh * dh:(hh + 1) * dh]
            ms = float(np.dot(uh, uh)) / dh * (3.0 * (hh + 1)) ** 2
            assert abs(math.sqrt(float(np.dot(kh, kh)) / dh) - 1.5 * math.sqrt(ms / (ms + EPS))) < 1e-12
            cos = float(np.dot(kh, uh)) / math.sqrt(float(np.dot(kh, kh)) * float(np.dot(uh, uh)))
            assert abs(cos - 1.0) < 1e-12


# ---------------------------------------------------------------- head (R12) + velocity wiring
def _head_expected(cfg, r, sh, sc, wh, bh):
    """v[c, f, i, j] by hand: token n = (f Hp + i//ph) Wp + j//pw, patch element
    p = ((c pt + 0) ph + i%ph) pw + j%pw (Conv3d flatten order, P9)."""
    C, F, Hh, Ww = cfg.latent_shape
    v = np.zeros(cfg.latent_shape)
    for c in range(C):
        for f in range(F):
            for i in range(Hh):
                for j in range(Ww):
                    n = (f * cfg.Hp + i // cfg.ph) * cfg.Wp + j // cfg.pw
                    p = ((c * cfg.pt) * cfg.ph + i % cfg.ph) * cfg.pw + j % cfg.pw
                    row = r[n]
                    ms = float(np.dot(row, row)) / cfg.d
                    hrow = row / math.sqrt(ms + EPS) * (1.0 + sc) + sh
                    v[c, f, i, j] = float(np.dot(hrow, wh[:, p])) + bh[p]
    return v


def test_head_shift_and_scale_rows():
    """(sh, sc) = head_mod + e, y = (RMSNorm(r)(1 + sc) + sh) W_h + b_h: shift-only and
    scale-only settings give different, hand-computable outputs (a swap, a dropped e or
    sc in place of 1 + sc fails)."""
    cfg = TINY
    P = OP.Params(cfg, 0)
    d, Pp = cfg.d, cfg.P
    r = np.zeros((cfg.N, d))
    r[:, 0] = 1.0
    r[:, 1] = 0.1 * np.arange(cfg.N)
    wh = np.zeros((d, Pp))
    wh[0, :] = np.arange(1, Pp + 1)
    wh[1, :] = 1.0
    bh = 0.05 * np.arange(Pp)
    P.set("head_w", wh); P.set("head_b", bh)
    # shift only: head_mod rows (0.3 - e, -e)
    e = np.full(d, 0.2)
    P.set("head_mod", np.stack([np.full(d, 0.1), np.full(d, -0.2)]))
    np.testing.assert_allclose(dit.head(P, cfg, r, e), _head_expected(cfg, r, 0.3, 0.0, wh, bh), rtol=0, atol=1e-12)
    # scale only: sh = 0, sc = 0.7
    P.set("head_mod", np.stack([np.full(d, -0.2), np.full(d, 0.5)]))
    np.testing.assert_allclose(dit.head(P, cfg, r, e), _head_expected(cfg, r, 0.0, 0.7, wh, bh), rtol=0, atol=1e-12)


def test_velocity_wires_patch_embed_and_e_into_head():
    """A zero-layer DiT: v = head(patchify(x) W_p + b_p, e_i) with e (not e6) conditioning the
    head.  W_p copies the patch into the first P columns (+ b_p = 0.1 everywhere); e6 is garbage
    and must not matter."""
    cfg = with_layers(TINY, 0)
    P = OP.Params(cfg, 0)
    d, Pp = cfg.d, cfg.P
    P.set("patch_w", _eye(cfg.P_in, d)); P.set("patch_b", np.full(d, 0.1))
    P.set("head_w", _eye(d, Pp, 1.0)); P.set("head_b", np.zeros(Pp))
    P.set("head_mod", np.stack([np.full(d, 0.1), np.full(d, 0.4)]))
    e = np.full(d, 0.05)
    cond = {"e": [None, e], "e6": [None, np.full((6, d), 1e3)], "kv": [], "kvi": None}
    x = np.random.default_rng(5).normal(size=cfg.latent_shape)
    v = dit.velocity(P, cfg, x, 1, cond)
    C, F, Hh, Ww = cfg.latent_shape
    for c in range(C):
        for f in range(F):
            for i in range(Hh):
                for j in range(Ww):
                    i0, j0 = i - i % cfg.ph, j - j % cfg.pw
                    patch = x[:, f, i0:i0 + cfg.ph, j0:j0 + cfg.pw]
                    ms = (float(np.sum((patch + 0.1) ** 2)) + (d - Pp) * 0.01) / d
                    want = (x[c, f, i, j] + 0.1) / math.sqrt(ms + EPS) * (1.0 + 0.45) + 0.15
                    assert abs(v[c, f, i, j] - want) < 1e-12


# ---------------------------------------------------------------- block wiring (R1, R3, R4, R9)
def _block_setup(cfg, g1, g2, co_zero=True):
    """Params for one block with q = k = 0 (uniform self-attention: o = mean_n v_n),
    v = h, o_w = I, and the cross-attention output projection zeroed; gates g1 / g2 come
    from the modulation table M_0 (e6 is passed separately)."""
    P = OP.Params(cfg, 0)
    d = cfg.d
    qkv = np.zeros((d, 3 * d))
    qkv[np.arange(d), 2 * d + np.arange(d)] = 1.0
    P.set("L0.qkv_w", qkv); P.set("L0.qkv_b", np.zeros(3 * d))
    P.set("L0.o_w", _eye(d, d)); P.set("L0.o_b", np.zeros(d))
    if co_zero:
        P.set("L0.co_w", np.zeros((d, d))); P.set("L0.co_b", np.zeros(d))
    mod = np.zeros((6, d))
    mod[2] = g1
    mod[5] = g2
    P.set("L0.mod", mod)
    return P, mod


def _alt_rows(cfg):
    a = 0.5 + 0.25 * np.arange(cfg.N)
    s = a / np.sqrt(a * a + EPS)                       # RMSNorm(a alt) = s alt, exactly
    return a[:, None] * _alt(cfg.d)[None, :], s


def _kv(cfg, seed=6):
    rr = np.random.default_rng(seed)
    return rr.normal(size=(cfg.L_txt, cfg.d)), rr.normal(size=(cfg.L_txt, cfg.d))


def test_self_attention_modulation_rows_0_1():
    """Row 0 of (e6 + M) shifts and row 1 scales the self-attention input:
    with uniform attention and v = h, r' = r + g1 mean_n h_n."""
    cfg = with_layers(TINY, 1)
    d = cfg.d
    r, s = _alt_rows(cfg)
    alt = _alt(d)
    c = np.linspace(-0.3, 0.4, d)
    pos = dit.token_positions(cfg)
    for which in ("shift", "scale"):
        P, mod = _block_setup(cfg, g1=0.5, g2=0.0)
        e6 = np.zeros((6, d))
        row = 0 if which == "shift" else 1
        e6[row] = 0.5 * c                       # half from e6, half from M_0: both must be added
        mod[row] = 0.5 * c
        P.set("L0.mod", mod)
        out = dit.block(P, cfg, 0, r, e6, _kv(cfg), pos)
        mean_h = s.mean() * alt + c if which == "shift" else s.mean() * alt * (1.0 + c)
        np.testing.assert_allclose(out, r + 0.5 * mean_h[None, :], rtol=0, atol=1e-12, err_msg=which)


def test_mlp_modulation_rows_3_4_and_swiglu_sides():
    """W1 = 0, b1 = 1, W3 = W2 = identity-like: a = SiLU(1) (h2 W3) is LINEAR in h2, so
    r' = r + g2 (SiLU(1) h2 + b2) with h2 = RMSNorm(r)(1 + sc2) + sh2 (rows 3/4 of e6 + M)."""
    cfg = with_layers(TINY, 1)
    d, f = cfg.d, cfg.ffn
    r, s = _alt_rows(cfg)
    alt = _alt(d)
    c = np.linspace(-0.3, 0.4, d)
    b2 = np.full(d, 0.07)
    pos = dit.token_positions(cfg)
    for which in ("shift", "scale"):
        P, mod = _block_setup(cfg, g1=0.0, g2=0.5)
        P.set("L0.w1", np.zeros((d, f))); P.set("L0.b1", np.ones(f))
        P.set("L0.w3", _eye(d, f)); P.set("L0.b3", np.zeros(f))
        P.set("L0.w2", _eye(f, d)); P.set("L0.b2", b2)
        e6 = np.zeros((6, d))
        row = 3 if which == "shift" else 4
        e6[row] = 0.5 * c
        mod[row] = 0.5 * c
        P.set("L0.mod", mod)
        out = dit.block(P, cfg, 0, r, e6, _kv(cfg), pos)
        h2 = s[:, None] * alt[None, :] + c if which == "shift" else s[:, None] * alt[None, :] * (1.0 + c)
        np.testing.assert_allclose(out, r + 0.5 * (_silu(1.0) * h2 + b2), rtol=0, atol=1e-12, err_msg=which)


def test_swiglu_silu_is_on_the_w1_branch():
    """W3 = 0, b3 = 1, W1 = W2 = identity-like: the MLP is SiLU(h2) -- nonlinear, odd-part
    free -- so r' = r + g2 SiLU(RMSNorm(r)) elementwise (SiLU on the W3 branch would give
    SiLU(1) h2 instead)."""
    cfg = with_layers(TINY, 1)
    d, f = cfg.d, cfg.ffn
    r, s = _alt_rows(cfg)
    alt = _alt(d)
    P, _ = _block_setup(cfg, g1=0.0, g2=0.5)
    P.set("L0.w1", _eye(d, f)); P.set("L0.b1", np.zeros(f))
    P.set("L0.w3", np.zeros((d, f))); P.set("L0.b3", np.ones(f))
    P.set("L0.w2", _eye(f, d)); P.set("L0.b2", np.zeros(d))
    out = dit.block(P, cfg, 0, r, np.zeros((6, d)), _kv(cfg), dit.token_positions(cfg))
    want = r + 0.5 * np.vectorize(_silu)(s[:, None] * alt[None, :])
    np.testing.assert_allclose(out, want, rtol=0, atol=1e-12)


def test_cross_attention_is_ungated_and_unmodulated():
    """Cross-attention with qc = 0 attends uniformly: its output is mean(V) W_co + b_co added
    to r with no gate and independently of the adaLN modulation (R3)."""
    cfg = with_layers(TINY, 1)
    d = cfg.d
    r, _ = _alt_rows(cfg)
    P, mod = _block_setup(cfg, g1=0.0, g2=0.0, co_zero=False)
    P.set("L0.cq_w", np.zeros((d, d))); P.set("L0.cq_b", np.zeros(d))
    bco = np.linspace(0, 0.2, d)
    P.set("L0.co_w", _eye(d, d, 2.0)); P.set("L0.co_b", bco)
    mod[0] = 5.0; mod[1] = -3.0; mod[3] = 7.0; mod[4] = 2.0        # modulation must not matter
    P.set("L0.mod", mod)
    kc, vc = _kv(cfg)
    out = dit.block(P, cfg, 0, r, np.zeros((6, d)), (kc, vc), dit.token_positions(cfg))
    np.testing.assert_allclose(out, r + (2.0 * vc.mean(axis=0) + bco)[None, :], rtol=0, atol=1e-12)


def test_cross_attention_query_path():
    """The cross query is headRMS((RMSNorm(r) g_n3) W_cq + b_cq) g_cq of the UNMODULATED
    residual (R3).  Two text keys k1 = kappa e_0, k2 = kappa e_1 per head split the softmax by
    the query's first two elements, which g_n3 (1.5 on even, 1 on odd elements) and the head
    norm fix: qc_even = 1.5 s / rms, qc_odd = -s / rms with rms = sqrt(3.25 s^2 / 2 + eps)."""
    cfg = with_layers(TINY, 1)
    d, H, dh = cfg.d, cfg.heads, cfg.dh
    r, s = _alt_rows(cfg)
    P, mod = _block_setup(cfg, g1=0.0, g2=0.0, co_zero=False)
    P.set("L0.g_n3", np.where(np.arange(d) % 2 == 0, 1.5, 1.0))
    P.set("L0.cq_w", _eye(d, d)); P.set("L0.cq_b", np.zeros(d)); P.set("L0.g_cq", np.ones(d))
    P.set("L0.co_w", _eye(d, d)); P.set("L0.co_b", np.zeros(d))
    mod[0] = 0.3; mod[1] = 0.6                                      # self-attn modulation: unused here
    P.set("L0.mod", mod)
    kappa = 3.0
    kc = np.zeros((2, d))
    kc[0, np.arange(H) * dh] = kappa
    kc[1, np.arange(H) * dh + 1] = kappa
    vc = np.random.default_rng(9).normal(size=(2, d))
    out = dit.block(P, cfg, 0, r, np.zeros((6, d)), (kc, vc), dit.token_positions(cfg))
    for n in range(cfg.N):
        sn = s[n]
        rms = math.sqrt(3.25 * sn * sn / 2.0 + EPS)
        q0, q1 = 1.5 * sn / rms, -sn / rms
        p1 = 1.0 / (1.0 + math.exp((q1 - q0) * kappa / math.sqrt(dh)))
        want = r[n] + p1 * vc[0] + (1.0 - p1) * vc[1]
        np.testing.assert_allclose(out[n], want, rtol=0, atol=1e-12)


# ---------------------------------------------------------------- encoder stand-in (R17)
def test_encoder_one_token_closed_form():
    """Embedding row a*alt, g_a = 1.5, W1 = W2 = identity-like, W3 = 2 I, g_f = 2:
    n = s alt (s = 1.5 a/sqrt(a^2+eps)), z_j = a alt_j + SiLU(n_j) 2 n_j, ctx = bf16(2 z/rms(z))."""
    cfg = TINY
    P = OP.Params(cfg, 0)
    dt, fe = cfg.d_txt, cfg.f_e
    a = 0.8
    emb = np.zeros((cfg.vocab, dt))
    emb[3] = a * _alt(dt)
    emb[5] = -a * _alt(dt)
    P.set("E.emb", emb)
    P.set("E.g_a", np.full(dt, 1.5)); P.set("E.g_f", np.full(dt, 2.0))
    P.set("E.e_w1", _eye(dt, fe)); P.set("E.e_w3", _eye(dt, fe, 2.0)); P.set("E.e_w2", _eye(fe, dt))
    ctx, bits = stages.encoder(P, cfg, np.array([3, 5, 3]))
    s = 1.5 * a / math.sqrt(a * a + EPS)
    zp = a + _silu(s) * 2 * s            # alt = +1
    zm = -a + _silu(-s) * (-2 * s)       # alt = -1
    rms = math.sqrt((zp * zp + zm * zm) / 2.0 + EPS)
    want3 = np.where(_alt(dt) > 0, 2 * zp / rms, 2 * zm / rms)
    want5 = np.where(_alt(dt) > 0, 2 * zm / rms, 2 * zp / rms)   # row 5 = -row 3: the signs swap
    for row, want in ((0, want3), (1, want5), (2, want3)):
        assert np.all(np.abs(ctx[row] - want) <= 2.0 ** -8 * np.abs(want)), (row, ctx[row][:4], want[:4])
    assert bits.dtype == np.uint16
