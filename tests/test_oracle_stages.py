"""Pins for the oracle's pipeline-level closed forms (Eq. 6, handoff hash,
chunking), the stand-in stages, and the vacuity guard."""
import math

import numpy as np
import pytest

from oracle import capacity as cap
from oracle import dit, stages
from oracle import params as OP
from synth.configs import TINY, MID, with_layers
from synth import inputs

# tab:stage_time, A10 Wan2.2 832x480: (Enc, DiT, Dec) seconds
T4 = (5.46, 74.1, 9.62)
T1 = (5.46, 18.7, 9.62)


@pytest.mark.parametrize("g,T,qpm,b", [
    ((1, 6, 1), T4, 4.858, "T"),    # P:L532 "4.9 QPM"
    ((1, 5, 2), T4, 4.049, "T"),    # P:L532 "4.0 QPM"
    ((1, 6, 1), T1, 6.237, "D"),    # P:L533 "6.2 QPM"
    ((1, 5, 2), T1, 10.989, "E"),   # P:L533 "11.0 QPM"
    ((1, 13, 2), T4, 10.526, "T"),  # P:L536 "10.5 QPM"
])
def test_eq6_paper_points(g, T, qpm, b):
    q, bott = cap.qps(g, T)
    assert abs(q * 60 - qpm) < 1e-3 and bott == b


def test_planner_exhaustive():
    assert cap.plan(8, T4) == (1, 6, 1)
    assert cap.plan(8, T1) == (2, 4, 2)      # SPEC S:L146 / SURVEY c.4 #28
    assert cap.plan(3, T4) == (1, 1, 1)
    for G in range(3, 13):
        best = cap.plan(G, T1)
        assert cap.feasible(best, G)
        q = cap.qps(best, T1)[0]
        for gE in range(1, G):
            for gT in range(1, G):
                for gD in range(1, G):
                    if cap.feasible((gE, gT, gD), G):
                        assert cap.qps((gE, gT, gD), T1)[0] <= q + 1e-12


def test_splitmix64_published_first_output():
    # splitmix64 seeded with 0: first output 0xE220A8397B1DCDAF (Steele, Lea, Flood 2014 / xoshiro seeding)
    assert int(cap.splitmix64(np.array([0], np.uint64))[0]) == 0xE220A8397B1DCDAF
    assert cap.payload_hash(bytes(8)) == 0xE220A8397B1DCDAF


def test_hash_chunk_additivity_and_order():
    buf = inputs.payload_bytes(1000, seed=1)     # not a multiple of 8 on purpose
    h = cap.payload_hash(buf)
    for chunk in (8, 64, 136, 512, 4096):
        parts = cap.chunks(1000, chunk)
        assert sum(s for _, s in parts) == 1000
        tot = 0
        for off, size in reversed(parts):        # any order
            tot = (tot + cap.payload_hash(buf[off:off + size], word_offset=off // 8)) % 2 ** 64
        assert tot == h
    buf2 = buf.copy(); buf2[500] ^= 1
    assert cap.payload_hash(buf2) != h
    # swapping two words changes the hash (position-keyed)
    w = buf[:16].copy(); w2 = np.concatenate([w[8:], w[:8]])
    assert cap.payload_hash(w) != cap.payload_hash(w2)


def test_jitter_rate():
    n = 4000
    hits = sum(cap.jitter_delayed(11, r, 0, 0.2) for r in range(n))
    assert abs(hits / n - 0.2) < 4 * math.sqrt(0.2 * 0.8 / n)
    assert not any(cap.jitter_delayed(11, r, 1, 0.0) for r in range(100))


def test_decoder_pixel_shuffle_bijection():
    # code every output index of D's second linear into its bias, zero weights:
    # o[idx] = tanh(artanh(code)) = code identifies idx; check every output lands where
    # the shuffle rule says and every output element is written exactly once.
    cfg = with_layers(MID, 1)
    cfg = type(cfg)(**{**cfg.__dict__, "F": 3})
    P = OP.Params(cfg, 0)
    for nm, r in (("D.d2f", 1), ("D.d2r", 4)):
        n = 3 * r * 64
        P.set(nm + "_w", np.zeros((cfg.dec_width, n)))
        P.set(nm + "_b", np.arctanh((np.arange(n) + 1) / (n + 2) * (1 if r == 1 else -1)))
    out = stages.decoder(P, cfg, np.zeros(cfg.latent_shape))
    assert out.shape == (3, 9, 8 * cfg.H, 8 * cfg.W)
    # frame 0 from d2f, frames 1..8 from d2r (tau = (t-1) % 4, phi = (t-1)//4 + 1)
    for t in range(9):
        r, n = (1, 192) if t == 0 else (4, 768)
        tau = 0 if t == 0 else (t - 1) % 4
        for ch in range(3):
            for dy in (0, 7):
                for dx in (0, 3):
                    idx = ((ch * r + tau) * 8 + dy) * 8 + dx
                    want = (idx + 1) / (n + 2) * (1 if r == 1 else -1)
                    assert abs(out[ch, t, 8 * 5 + dy, 8 * 9 + dx] - want) < 1e-12


def test_encoder_payload_is_bf16_and_normalised():
    P = OP.Params(TINY, 0)
    ctx, bits = stages.encoder(P, TINY, stages.tokens_from_seed(TINY, 1))
    assert bits.dtype == np.uint16 and ctx.shape == (TINY.L_txt, TINY.d_txt)
    np.testing.assert_array_equal(OP.bf16_bits_to_f64(bits), ctx)
    rms = np.sqrt(np.mean((ctx / P["E.g_f"]) ** 2, axis=-1))
    np.testing.assert_allclose(rms, 1.0, rtol=2e-2)


def _vacuity(cfg, seed=0):
    P = OP.Params(cfg, 0)
    sig = dit.sigmas(cfg.steps, cfg.shift)
    ctx = inputs.bf16_bits_to_f64(inputs.ctx_bf16(cfg, seed))
    cond = dit.prologue(P, cfg, ctx, sig)
    x = inputs.latent(cfg, seed).astype(np.float64)
    tr = []
    v = dit.velocity(P, cfg, x, 1, cond, trace=tr)
    rho = [np.linalg.norm(tr[l + 1] - tr[l]) / np.linalg.norm(tr[l]) for l in range(cfg.layers)]
    v0 = dit.velocity(P, cfg, x, 1, cond, cross=False)
    return rho, np.linalg.norm(v) / np.linalg.norm(x), np.linalg.norm(v - v0) / np.linalg.norm(v)


@pytest.mark.parametrize("cfg", [TINY, MID])
def test_vacuity_guard(cfg):
    rho, vx, dcross = _vacuity(cfg)
    assert all(1e-2 <= r <= 1.0 for r in rho), rho
    assert 0.1 <= vx <= 10.0, vx
    assert dcross >= 5e-2, dcross


@pytest.mark.parametrize("name", ["image", "video"])
def test_vacuity_guard_production_width(name):
    """The guard at the C2 / C3 widths (d, heads, f, L_txt, the weights' std table) on one
    latent frame of 16x16 (N = 64) and one block; the full depths (28 / 40 blocks) are run
    by tools/vacuity_full_depth.py (profiles/r02_vacuity_*_full_depth.json)."""
    import dataclasses
    from synth.configs import CONFIGS
    cfg = dataclasses.replace(with_layers(CONFIGS[name], 1), F=1, H=16, W=16)
    rho, vx, dcross = _vacuity(cfg)
    assert all(1e-2 <= r <= 1.0 for r in rho), rho
    assert 0.1 <= vx <= 10.0, vx
    assert dcross >= 5e-2, dcross


def test_pipeline_request_tiny_runs():
    P = OP.Params(TINY, 0)
    out = stages.request(P, TINY, seed=1)
    assert out["latent"].dtype == np.float32 and np.all(np.isfinite(out["out"]))
    assert out["out"].shape == TINY.out_shape


def test_planner_move_budget_spec_example():
    # 1-step stage times, current (1,6,1), <= 2 instance moves -> (1,5,2)
    assert cap.plan(8, T1, cur=(1, 6, 1), budget=2) == (1, 5, 2)
    assert cap.plan(8, T1) == (2, 4, 2)                   # unconstrained optimum differs (R25)
    assert cap.plan(8, T4, cur=(1, 5, 2), budget=8) == (1, 6, 1)


def test_reactive_rule_spec_examples():
    # S:L489-491
    assert cap.reactive(0.95, 7, 4.8, 3.1, 6, 8 - 1, 8) == 1       # ScaleOut(T), one GPU free
    assert cap.reactive(0.95, 7, 4.8, 3.1, 6, 8, 8) == 0           # no free GPU: capacity
    assert cap.reactive(0.10, 0, 0.0, 0.0, 2, 8, 8) == -1          # ScaleIn(D)
    assert cap.reactive(0.10, 0, 0.0, 0.0, 1, 8, 8) == 0           # never below one instance
    assert cap.reactive(0.50, 2, 1.0, 0.5, 1, 8, 8) == 0           # NoOp
    assert cap.reactive(0.95, 7, 4.8, None, 6, 7, 8) == 0          # first tick: no d'


def test_change_detector_spec_examples():
    assert not cap.changed([4] * 20)
    assert cap.changed([4] * 15 + [1] * 5)
    assert not cap.changed([4] * 12 + [1, 1, 4, 4])   # tie in the recent window -> no change


def test_image_encoder_stand_in_invariants():
    """I2V E stand-in (R27): unit-variance uniform tokens bounded by sqrt(3), the first-frame
    mask exactly 1 on latent frame 0 and y zero on later frames, seed-determined."""
    from synth.configs import TINY_I2V, MID_I2V
    cfg = MID_I2V
    clip_bits, y = stages.image_encoder(cfg, 11)
    clip = (clip_bits.astype(np.uint32) << np.uint32(16)).view(np.float32).astype(np.float64)
    assert clip.shape == (cfg.L_img, cfg.d_img) and y.shape == cfg.y_shape and y.dtype == np.float32
    assert np.abs(clip).max() <= np.sqrt(3.0) * (1 + 2 ** -8)
    n = clip.size
    assert abs(clip.mean()) < 5 / np.sqrt(n) and abs(clip.var() - 1.0) < 0.05
    assert np.all(y[:4, 0] == 1.0) and np.all(y[:, 1:] == 0.0)
    lat = y[4:, 0].astype(np.float64)
    assert abs(lat.mean()) < 5 / np.sqrt(lat.size) and abs(lat.var() - 1.0) < 0.05
    c2, y2 = stages.image_encoder(cfg, 11)
    c3, y3 = stages.image_encoder(cfg, 12)
    assert np.array_equal(c2, clip_bits) and np.array_equal(y2, y)
    assert not np.array_equal(c3, clip_bits) and not np.array_equal(y3, y)
    ct, yt = stages.image_encoder(TINY_I2V, 11)
    assert ct.shape == (TINY_I2V.L_img, TINY_I2V.d_img) and yt.shape == TINY_I2V.y_shape
