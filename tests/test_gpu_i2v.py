"""Image-to-video conditioning (NEXT-3; R27) against the fp64
oracle: the patch embedding reads concat(x, y) and every block adds a cross-attention
over the image tokens.  Same tolerances as the text-to-video path (BASELINE.json
north_star): one bf16 step rel-L2 <= 1e-2, a trajectory <= 3e-2, fp32 build <= 1e-4."""
import numpy as np
import pytest

from oracle import params as OP, dit
from synth import inputs
from synth.configs import TINY_I2V, MID_I2V
from gpu_util import rel_l2, bf16_tensor_from_bits, make_ctx

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

BF16, FP32 = 0, 1
TOL_STEP = {BF16: 1e-2, FP32: 1e-4}
TOL_TRAJ = {BF16: 3e-2, FP32: 1e-4}


def _inputs(cfg, seed):
    return (inputs.latent(cfg, seed), inputs.ctx_bf16(cfg, seed + 1), inputs.clip_bf16(cfg, seed + 2),
            inputs.y_cond(cfg, seed + 3))


def _oracle_cond(P, cfg, ctx_bits, clip_bits, y, sig):
    return dit.prologue(P, cfg, inputs.bf16_bits_to_f64(ctx_bits), sig, clip=inputs.bf16_bits_to_f64(clip_bits),
                        y=y.astype(np.float64))


def test_i2v_weight_bits():
    """Parity check 0 for the I2V tensors: the wider patch embedding and the image paths."""
    cfg = TINY_I2V
    P = OP.Params(cfg, 7)
    with make_ctx(cfg, seed=7) as c:
        for name in ("patch_w", "img1_w", "img2_b", "L0.ki_w", "L1.vi_w", "L1.vi_b", "L0.g_ki"):
            got = c.weight_bits(1, P.tid(name), int(np.prod(P[name].shape)))
            assert np.array_equal(got, P.bits(name).reshape(-1)), name


@pytest.mark.parametrize("prec", [BF16, FP32])
@pytest.mark.parametrize("cfg,i", [(TINY_I2V, 0), (TINY_I2V, 3), (MID_I2V, 2)])
def test_i2v_step_parity(cfg, i, prec):
    x, ctx_bits, clip_bits, y = _inputs(cfg, 30)
    sig = dit.sigmas(cfg.steps, cfg.shift).astype(np.float32)
    with make_ctx(cfg, precision=prec) as c:
        cond = c.dit_prepare_i2v(1, bf16_tensor_from_bits(ctx_bits), bf16_tensor_from_bits(clip_bits),
                                 torch.from_numpy(y).cuda(), sig)
        xt = torch.from_numpy(x).cuda()
        vt = torch.zeros_like(xt)
        c.dit_step(1, cond, i, xt, vt)
        torch.cuda.synchronize()
        c.cond_release(cond)
        gx, gv = xt.cpu().numpy(), vt.cpu().numpy()
    P = OP.Params(cfg, 0)
    sig64 = sig.astype(np.float64)
    ox, ov = dit.step(P, cfg, x.astype(np.float64), i, _oracle_cond(P, cfg, ctx_bits, clip_bits, y, sig64), sig64)
    assert rel_l2(gv, ov) <= TOL_STEP[prec], rel_l2(gv, ov)
    assert rel_l2(gx, ox) <= TOL_STEP[prec]


@pytest.mark.parametrize("prec", [BF16, FP32])
def test_i2v_trajectory_parity(prec):
    cfg = TINY_I2V
    x0, ctx_bits, clip_bits, y = _inputs(cfg, 40)
    sig = dit.sigmas(cfg.steps, cfg.shift).astype(np.float32)
    with make_ctx(cfg, precision=prec) as c:
        cond = c.dit_prepare_i2v(1, bf16_tensor_from_bits(ctx_bits), bf16_tensor_from_bits(clip_bits),
                                 torch.from_numpy(y).cuda(), sig)
        xt = torch.from_numpy(x0).cuda()
        for i in range(cfg.steps):
            c.dit_step(1, cond, i, xt)
        torch.cuda.synchronize()
        c.cond_release(cond)
        gx = xt.cpu().numpy()
    P = OP.Params(cfg, 0)
    ox = dit.trajectory(P, cfg, x0.astype(np.float64), inputs.bf16_bits_to_f64(ctx_bits),
                        clip=inputs.bf16_bits_to_f64(clip_bits), y=y.astype(np.float64))
    assert rel_l2(gx, ox) <= TOL_TRAJ[prec], rel_l2(gx, ox)


def test_i2v_cfg_step_parity():
    """I2V with classifier-free guidance: the negative sample keeps the image conditioning."""
    cfg = TINY_I2V
    x, ctx_bits, clip_bits, y = _inputs(cfg, 50)
    neg_bits = inputs.ctx_bf16(cfg, 55)
    g = 4.0
    sig = dit.sigmas(cfg.steps, cfg.shift).astype(np.float32)
    with make_ctx(cfg) as c:
        cond = c.dit_prepare_i2v(1, bf16_tensor_from_bits(ctx_bits), bf16_tensor_from_bits(clip_bits),
                                 torch.from_numpy(y).cuda(), sig, ctx_neg_dev=bf16_tensor_from_bits(neg_bits),
                                 guidance=g)
        xt = torch.from_numpy(x).cuda()
        vt = torch.zeros_like(xt)
        c.dit_step(1, cond, 1, xt, vt)
        torch.cuda.synchronize()
        c.cond_release(cond)
        gv = vt.cpu().numpy()
    P = OP.Params(cfg, 0)
    sig64 = sig.astype(np.float64)
    cc = _oracle_cond(P, cfg, ctx_bits, clip_bits, y, sig64)
    cn = _oracle_cond(P, cfg, neg_bits, clip_bits, y, sig64)
    ov = dit.velocity_cfg(P, cfg, x.astype(np.float64), 1, cc, cn, g)
    assert rel_l2(gv, ov) <= TOL_STEP[BF16], rel_l2(gv, ov)


def test_i2v_needs_image_inputs():
    """The text-only prologue refuses an I2V graph (it has no image inputs)."""
    from paper_2605_25550_b200.binding import DFError
    cfg = TINY_I2V
    ctx_bits = inputs.ctx_bf16(cfg, 60)
    with make_ctx(cfg) as c:
        with pytest.raises(DFError):
            c.dit_prepare(1, bf16_tensor_from_bits(ctx_bits), dit.sigmas(cfg.steps, cfg.shift).astype(np.float32))


def test_i2v_image_encoder_equals_oracle():
    """The E stand-in's image conditioning (clip bf16, y fp32) is bit-exact with the oracle's."""
    from oracle import stages
    from synth.configs import TINY_I2V
    cfg = TINY_I2V
    with make_ctx(cfg) as c:
        clip = torch.zeros((cfg.L_img, cfg.d_img), device="cuda", dtype=torch.bfloat16)
        y = torch.zeros(cfg.y_shape, device="cuda")
        c.image_cond(0, 987, clip, y)
        torch.cuda.synchronize()
        want_clip, want_y = stages.image_encoder(cfg, 987)
        got_clip = clip.view(torch.int16).cpu().numpy().view(np.uint16)
        assert np.array_equal(got_clip, want_clip)
        assert np.array_equal(y.cpu().numpy(), want_y)


@pytest.mark.parametrize("guidance", [1.0, 3.0])
def test_i2v_pipeline_matches_oracle(guidance):
    """E -> T -> D with the image conditioning in the E->T payload ([ctx | clip | y | ctx_neg],
    chunked, hashed): outputs within the trajectory tolerance of the serial oracle request."""
    from oracle import stages, capacity as cap
    from paper_2605_25550_b200 import binding as B
    cfg = TINY_I2V
    P = OP.Params(cfg, 0)
    seeds = [5, 6]
    with make_ctx(cfg, handoff_mode=B.DF_ASYNC | B.DF_HASH, chunk_bytes=(96, 256)) as c:
        outs = {s: np.zeros(cfg.out_shape, np.float32) for s in seeds}
        for s in seeds:
            st, _ = c.submit(cfg.steps, cfg.shift, s, out_host=outs[s], user_tag=s, guidance=guidance)
            assert st == B.DF_OK
        comps = []
        while len(comps) < len(seeds):
            comps += c.poll(16, timeout_ms=60000)
    assert sorted(x.user_tag for x in comps) == seeds
    for x in comps:
        for e in range(2):
            assert x.hash_src[e] == x.hash_dst[e] != 0
        want = stages.request(P, cfg, seed=int(x.user_tag), guidance=guidance)
        assert rel_l2(outs[x.user_tag], want["out"]) <= 3e-2


def test_i2v_layer_parity_production_widths():
    """One I2V block at the video model's widths (d = 5120, 40 heads, 257 image tokens of
    width 1280 -> 3 key blocks with a ragged tail, C_y = 20 -> a 144-wide patch input) on a
    2-frame 480x832 latent, 64 sampled rows plus the ragged last rows, vs oracle.block_rows."""
    import dataclasses
    from synth.configs import VIDEO_I2V, with_layers
    cfg = dataclasses.replace(with_layers(VIDEO_I2V, 1), F=2)
    x_r = inputs.residual(cfg, 71)
    ctx_bits, clip_bits, y = inputs.ctx_bf16(cfg, 72), inputs.clip_bf16(cfg, 73), inputs.y_cond(cfg, 74)
    sig = dit.sigmas(cfg.steps, cfg.shift).astype(np.float32)
    i = 5
    rows = np.concatenate([np.sort(np.random.default_rng(2).choice(cfg.N - 40, 48, replace=False)),
                           np.arange(cfg.N - 16, cfg.N)])
    with make_ctx(cfg) as c:
        cond = c.dit_prepare_i2v(1, bf16_tensor_from_bits(ctx_bits), bf16_tensor_from_bits(clip_bits),
                                 torch.from_numpy(y).cuda(), sig)
        rt = torch.from_numpy(x_r).cuda()
        c.dit_layer(1, cond, i, 0, rt)
        torch.cuda.synchronize()
        c.cond_release(cond)
        got = rt.cpu().numpy()[rows]
    P = OP.Params(cfg, 0)
    kv = dit.cross_kv(P, cfg, 0, dit.text_projection(P, cfg, inputs.bf16_bits_to_f64(ctx_bits)))
    kvi = dit.image_kv(P, cfg, 0, dit.image_projection(P, cfg, inputs.bf16_bits_to_f64(clip_bits)))
    _, e6 = dit.time_embedding(P, cfg, float(sig[i]))
    want = dit.block_rows(P, cfg, 0, x_r.astype(np.float64), e6, kv, dit.token_positions(cfg), rows, kvi=kvi)
    assert rel_l2(got - x_r[rows], want - x_r[rows]) <= 1e-2
