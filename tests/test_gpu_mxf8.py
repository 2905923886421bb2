"""NEXT-4 MXFP8 parity (R30): the OCP MX quantiser (bit-exact e4m3 codes and E8M0
scale bytes) and the block-scaled CTA-pair GEMM (tcgen05 kind::mxf8f6f4.block_scale) against
oracle/fp8.py, through the C ABI.

The scale bytes come back in the tiled layout df.h documents; `_untile` below is that layout
written out (test code), so a wrong atom or byte order in either the quantiser or the GEMM's
TMEM copy shows up as a mismatch."""
import numpy as np
import pytest
import torch

from oracle import fp8
from synth import inputs
from synth.configs import TINY
from gpu_util import bf16_tensor_from_bits, make_ctx

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    with make_ctx(TINY) as c:
        yield c


def _sf_bytes(M, K):
    return (K // 128) * ((M + 127) // 128) * 512


def _tile_index(M, K):
    """Byte offset of scale (row m, k-block kb) in df.h's tiled layout, for all m < M, kb < K/32."""
    RB = (M + 127) // 128
    m = np.arange(M)[:, None]
    kb = np.arange(K // 32)[None, :]
    return ((kb // 4) * RB + m // 128) * 512 + (m % 32) * 16 + ((m % 128) // 32) * 4 + kb % 4


def _untile(sf, M, K):
    return np.asarray(sf)[_tile_index(M, K)]


def _tile(sbytes, M, K):
    out = np.zeros(_sf_bytes(M, K), np.uint8)
    out[_tile_index(M, K)] = sbytes
    return out


def _quant_gpu(ctx, bits):
    M, K = bits.shape
    x = bf16_tensor_from_bits(bits)
    q = torch.full((M, K), 0xAB, dtype=torch.uint8, device="cuda")
    sf = torch.full((_sf_bytes(M, K),), 0xCD, dtype=torch.uint8, device="cuda")
    ctx.op_mx_quant_e4m3(x, q, sf)
    torch.cuda.synchronize()
    return q.cpu().numpy(), sf.cpu().numpy()


@pytest.mark.parametrize("M,K", [(1, 128), (256, 128), (300, 3072), (4096, 3072), (130, 8192)])
def test_mx_quant_bit_exact(ctx, M, K):
    bits = inputs.activation_bf16((M, K), seed=M * 7 + K)
    q, sf = _quant_gpu(ctx, bits)
    q_ref, s_ref = fp8.mx_quantize(inputs.bf16_bits_to_f64(bits))
    assert np.array_equal(q, q_ref)
    assert np.array_equal(_untile(sf, M, K), s_ref)
    # rows past M in the last 128-row block carry scale byte 0
    pad = np.ones(_sf_bytes(M, K), bool)
    pad[_tile_index(M, K)] = False
    assert not sf[pad].any()


def test_mx_quant_wide_exponent_range(ctx):
    """Blocks spanning 2^-100 .. 2^100 (incl. bf16 subnormal and zero blocks)."""
    M, K = 256, 256
    r = np.random.default_rng(3)
    x = r.standard_normal((M, K)) * np.exp2(r.integers(-100, 100, size=(M, K // 32))).repeat(32, axis=1)
    x[5, 32:64] = 0.0
    x[7, :32] = 2.0 ** -133  # smallest bf16 subnormal
    bits = inputs.f32_to_bf16_bits_trunc(x.astype(np.float32))
    q, sf = _quant_gpu(ctx, bits)
    q_ref, s_ref = fp8.mx_quantize(inputs.bf16_bits_to_f64(bits))
    assert np.array_equal(q, q_ref)
    assert np.array_equal(_untile(sf, M, K), s_ref)


def _gemm_gpu(ctx, qa, sa, qb, sb, out_dtype=torch.float32):
    M, K = qa.shape
    N = qb.shape[0]
    out = torch.full((M, N), float("nan"), dtype=out_dtype, device="cuda")
    ctx.op_gemm_mxf8(torch.from_numpy(qa).cuda(), torch.from_numpy(_tile(sa, M, K)).cuda(),
                     torch.from_numpy(qb).cuda(), torch.from_numpy(_tile(sb, N, K)).cuda(), out)
    torch.cuda.synchronize()
    return out.float().cpu().numpy().astype(np.float64)


@pytest.mark.parametrize("M,N,K", [(256, 256, 128), (512, 768, 1024), (300, 520, 384)])
def test_mx_gemm_exact_on_small_integers(ctx, M, N, K):
    """Small-integer codes with per-block scales 2^-2 .. 2^2 (every scale byte differs from its
    neighbours): every product and partial sum is exact in fp32, so the tensor-core result must
    equal the fp64 oracle bit for bit -- a scale applied to the wrong row, column or k-block,
    or a wrong byte of a TMEM scale column, cannot hide."""
    r = np.random.default_rng(M + N + K)
    ints = np.array([0, 1, 2, 3, 4, 6, 8], dtype=np.float64)
    a = r.choice(ints, size=(M, K)) * r.choice([-1.0, 1.0], size=(M, K))
    b = r.choice(ints, size=(N, K)) * r.choice([-1.0, 1.0], size=(N, K))
    qa, qb = fp8.e4m3_encode(a), fp8.e4m3_encode(b)
    sa = (127 + r.integers(-2, 3, size=(M, K // 32))).astype(np.uint8)
    sb = (127 + r.integers(-2, 3, size=(N, K // 32))).astype(np.uint8)
    got = _gemm_gpu(ctx, qa, sa, qb, sb)
    want = fp8.gemm_mxf8(qa, sa, qb, sb)
    assert np.array_equal(got, want), f"max |err| {np.max(np.abs(got - want))}"


@pytest.mark.parametrize("M,N,K", [(512, 512, 1024), (4096, 3072, 3072), (4096, 12288, 3072), (1000, 2000, 8192)])
def test_mx_gemm_vs_oracle_realistic(ctx, M, N, K):
    """bf16 activations / weights quantised on the GPU (bit-exact above), GEMM against the fp64
    oracle within the fp32 accumulation bound 2^-17 sum|a||b| (as R28's per-tensor GEMM)."""
    abits = inputs.activation_bf16((M, K), seed=M + K)
    bbits = inputs.activation_bf16((N, K), seed=N + K + 1, outlier_frac=0.0)
    qa_t = torch.empty((M, K), dtype=torch.uint8, device="cuda")
    qb_t = torch.empty((N, K), dtype=torch.uint8, device="cuda")
    sa_t = torch.empty((_sf_bytes(M, K),), dtype=torch.uint8, device="cuda")
    sb_t = torch.empty((_sf_bytes(N, K),), dtype=torch.uint8, device="cuda")
    ctx.op_mx_quant_e4m3(bf16_tensor_from_bits(abits), qa_t, sa_t)
    ctx.op_mx_quant_e4m3(bf16_tensor_from_bits(bbits), qb_t, sb_t)
    out = torch.full((M, N), float("nan"), device="cuda")
    ctx.op_gemm_mxf8(qa_t, sa_t, qb_t, sb_t, out)
    torch.cuda.synchronize()
    qa, sa = fp8.mx_quantize(inputs.bf16_bits_to_f64(abits))
    qb, sb = fp8.mx_quantize(inputs.bf16_bits_to_f64(bbits))
    want = fp8.gemm_mxf8(qa, sa, qb, sb)
    bound = np.abs(fp8.mx_dequantize(qa, sa)) @ np.abs(fp8.mx_dequantize(qb, sb)).T
    got = out.cpu().numpy().astype(np.float64)
    assert np.all(np.isfinite(got))
    print("mxf8 gemm", M, N, K, "max |err|/bound = %.3g" % float(np.max(np.abs(got - want) / np.maximum(bound, 1e-300))))
    assert np.all(np.abs(got - want) <= 2.0 ** -17 * bound + 1e-30)
    if M * N * K > 1e10:
        return
    # the e4m3 element error itself: a few % of the bf16 product (3 mantissa bits; R30's OCP
    # floor scale also saturates the largest element of ~1/5 of the blocks)
    exact = inputs.bf16_bits_to_f64(abits) @ inputs.bf16_bits_to_f64(bbits).T
    e_mx = np.linalg.norm(got - exact) / np.linalg.norm(exact)
    print("rel-L2 vs the bf16 product: MXFP8 %.3g" % e_mx)
    assert e_mx < 6e-2


def test_mx_block_scales_keep_a_wide_dynamic_range(ctx):
    """What block scaling buys over one scale per tensor: activation rows whose magnitudes span
    2^-20 .. 2^4.  Per-tensor e4m3 pushes the small rows into e4m3 subnormals / zero; MXFP8
    keeps every block at full relative precision."""
    M, N, K = 512, 512, 1024
    r = np.random.default_rng(21)
    a = r.standard_normal((M, K)) * np.exp2(r.integers(-20, 5, size=(M, 1)))
    abits = inputs.f32_to_bf16_bits_trunc(a.astype(np.float32))
    bbits = inputs.activation_bf16((N, K), seed=22, outlier_frac=0.0)
    af, bf = inputs.bf16_bits_to_f64(abits), inputs.bf16_bits_to_f64(bbits)
    qa, sa = fp8.mx_quantize(af)
    qb, sb = fp8.mx_quantize(bf)
    got = _gemm_gpu(ctx, qa, sa, qb, sb)
    exact = af @ bf.T
    pa, s1 = fp8.quantize_per_tensor(af.astype(np.float32))
    pb, s2 = fp8.quantize_per_tensor(bf.astype(np.float32))
    per_tensor = fp8.gemm_e4m3(pa, pb, s1, s2)
    # per row: the rows dominated by small blocks are where per-tensor scaling fails
    e_mx = np.linalg.norm(got - exact, axis=1) / np.linalg.norm(exact, axis=1)
    e_pt = np.linalg.norm(per_tensor - exact, axis=1) / np.linalg.norm(exact, axis=1)
    print("per-row rel-L2, median / max: MXFP8 %.3g / %.3g, per-tensor %.3g / %.3g"
          % (np.median(e_mx), e_mx.max(), np.median(e_pt), e_pt.max()))
    assert e_mx.max() < 6e-2 and e_pt.max() > 2 * e_mx.max()


def test_mx_gemm_bf16_out(ctx):
    r = np.random.default_rng(9)
    a = r.standard_normal((512, 512))
    b = r.standard_normal((256, 512))
    qa, sa = fp8.mx_quantize(a)
    qb, sb = fp8.mx_quantize(b)
    got = _gemm_gpu(ctx, qa, sa, qb, sb, torch.bfloat16)
    want = fp8.gemm_mxf8(qa, sa, qb, sb)
    bound = np.abs(fp8.mx_dequantize(qa, sa)) @ np.abs(fp8.mx_dequantize(qb, sb)).T
    assert np.all(np.abs(got - want) <= 2.0 ** -8 * np.abs(want) + 2.0 ** -17 * bound + 1e-30)


def test_mx_rejects_bad_shapes(ctx):
    from paper_2605_25550_b200 import binding as B
    x = torch.zeros((256, 96), dtype=torch.bfloat16, device="cuda")  # K % 128 != 0
    with pytest.raises(B.DFError):
        ctx.op_mx_quant_e4m3(x, torch.empty((256, 96), dtype=torch.uint8, device="cuda"),
                             torch.empty(4096, dtype=torch.uint8, device="cuda"))
    q = torch.zeros((256, 96), dtype=torch.uint8, device="cuda")
    with pytest.raises(B.DFError):
        ctx.op_gemm_mxf8(q, torch.zeros(4096, dtype=torch.uint8, device="cuda"), q,
                         torch.zeros(4096, dtype=torch.uint8, device="cuda"), torch.empty((256, 256), device="cuda"))


# ---------------------------------------------------------------- MXFP8 step mode (R31)
TOL_MX_STEP = 2.5e-2  # DESIGN.md R31 (R29's code-flip argument, with MX's finer scales)


@pytest.mark.parametrize("i", [0, 5])
def test_mxfp8_step_matches_the_mx_oracle(i):
    """NEXT-4 in the DiT step with MXFP8 operands (R31): all six block GEMMs block-scaled
    (activations by the RMSNorm / MX quantiser, weights at init), the rest bf16.  Against the
    fp64 oracle of the same mode within R31's tolerance; against the bf16 oracle it differs by
    the quantisation itself (so the mode is not a silent bf16 or per-row FP8 run)."""
    from oracle import dit, dit_fp8
    from oracle import params as OP
    from synth.configs import MID
    from gpu_util import rel_l2
    from paper_2605_25550_b200 import binding as B
    cfg = MID
    x = inputs.latent(cfg, 91)
    ctx_bits = inputs.ctx_bf16(cfg, 92)
    sig = dit.sigmas(cfg.steps, cfg.shift).astype(np.float32)
    with make_ctx(cfg, precision=B.DF_MXFP8) as c:
        cond = c.dit_prepare(1, bf16_tensor_from_bits(ctx_bits), sig)
        xt = torch.from_numpy(x).cuda()
        vt = torch.zeros_like(xt)
        c.dit_step(1, cond, i, xt, vt)
        torch.cuda.synchronize()
        c.cond_release(cond)
        gx, gv = xt.cpu().numpy(), vt.cpu().numpy()
    P = OP.Params(cfg, 0)
    sig64 = sig.astype(np.float64)
    cond = dit.prologue(P, cfg, inputs.bf16_bits_to_f64(ctx_bits), sig64)
    oxm, ovm = dit_fp8.step_mx(P, cfg, x.astype(np.float64), i, cond, sig64)
    ox8, ov8 = dit_fp8.step(P, cfg, x.astype(np.float64), i, cond, sig64)
    ox, ov = dit.step(P, cfg, x.astype(np.float64), i, cond, sig64)
    err, q_err, r29 = rel_l2(gv, ovm), rel_l2(ovm, ov), rel_l2(ov8, ov)
    print(f"mxfp8 step i={i}: GPU vs MX oracle {err:.3e}; MX oracle vs bf16 oracle {q_err:.3e} "
          f"(per-row FP8 oracle vs bf16 oracle {r29:.3e})")
    assert err <= TOL_MX_STEP, err
    assert rel_l2(gx, oxm) <= TOL_MX_STEP
    assert err < q_err < 0.2, (err, q_err)
    assert rel_l2(gv, ov8) > err  # closer to its own mode's oracle than to the per-row FP8 mode's


def test_mxfp8_pipeline_deterministic():
    """The MXFP8 mode through the serving API: two identical requests give identical bytes."""
    from synth.configs import MID
    from paper_2605_25550_b200 import binding as B
    cfg = MID
    ctx_bits = inputs.ctx_bf16(cfg, 5)
    outs = []
    with make_ctx(cfg, precision=B.DF_MXFP8) as c:
        from oracle import dit as odit
        s = odit.sigmas(cfg.steps, cfg.shift).astype(np.float32)
        for _ in range(2):
            cond = c.dit_prepare(1, bf16_tensor_from_bits(ctx_bits), s)
            xt = torch.from_numpy(inputs.latent(cfg, 6)).cuda()
            for i in range(3):
                c.dit_step(1, cond, i, xt)
            torch.cuda.synchronize()
            c.cond_release(cond)
            outs.append(xt.cpu().numpy())
    assert np.array_equal(outs[0], outs[1])
    assert np.isfinite(outs[0]).all()
