"""Mutation check of the oracle's pins (VERDICT r1 "Next round" #1): every plausible
one-line misreading of an oracle function must fail at least one `-m "not gpu"` pin.

    python tools/mutate_oracle.py [--log profiles/r02_oracle_mutations.txt] [-j 8]

Each mutation copies oracle/, synth/ and the oracle pin tests to a scratch directory,
applies ONE textual replacement to the copy, and runs the pin tests there; the mutation is
"killed" when pytest fails.  The unmutated copy must pass (sanity).  Test infrastructure
only: it reads oracle/ as text and never imports the product package.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TESTS = ["tests/test_oracle_pins.py", "tests/test_oracle_math.py", "tests/test_oracle_stages.py",
         "tests/test_oracle_rng.py", "tests/test_oracle_fp8.py"]

# (id, file, old, new, what it models)
MUTATIONS = [
    # ---- FP8 / MXFP8 (R28-R33), added with the MXFP8 and FP8-attention oracles
    ("mx-emax-7", "oracle/fp8.py", "- E4M3_EMAX\n", "- E4M3_EMAX + 1\n", "MX scale exponent with emax 7"),
    ("mx-ceil", "oracle/fp8.py", "e = np.floor(np.log2(np.where(amax > 0, amax, 1.0))) - E4M3_EMAX",
     "e = np.ceil(np.log2(np.where(amax > 0, amax, 1.0))) - E4M3_EMAX", "ceil instead of OCP's floor"),
    ("mx-zero-block-e0", "oracle/fp8.py", "e = np.where(amax > 0, e, -127.0)", "e = np.where(amax > 0, e, 0.0)",
     "zero block with scale byte 127"),
    ("mx-bias-126", "oracle/fp8.py", "sc = np.exp2(np.asarray(sbytes, dtype=np.float64) - 127.0)",
     "sc = np.exp2(np.asarray(sbytes, dtype=np.float64) - 126.0)", "E8M0 bias off by one"),
    ("mx-weight-blocks-along-n", "oracle/dit_fp8.py",
     "q, s = fp8.mx_quantize(np.asarray(W, dtype=np.float64).T)\n    return fp8.mx_dequantize(q, s).T",
     "q, s = fp8.mx_quantize(np.asarray(W, dtype=np.float64))\n    return fp8.mx_dequantize(q, s)",
     "MX weight blocks along N instead of K"),
    ("qk-scale-no-sqrt-dh", "oracle/dit_fp8.py", "np.sqrt(float(dh)) * gmax / 448.0", "gmax / 448.0",
     "Q/K scale without the sqrt(dh) bound"),
    ("qk-scale-not-pow2", "oracle/dit_fp8.py",
     "return pow2_ceil(np.float32(np.sqrt(float(dh)) * gmax / 448.0)) if gmax > 0 else np.float32(1.0)",
     "return np.float32(np.sqrt(float(dh)) * gmax / 448.0) if gmax > 0 else np.float32(1.0)",
     "Q/K scale not rounded to a power of two"),
    ("v-scale-not-pow2", "oracle/dit_fp8.py",
     "s = pow2_ceil(np.float32(amax / E4M3_MAX)) if amax > 0 else np.float32(1.0)\n    return fp8.e4m3_decode",
     "s = np.float32(amax / E4M3_MAX) if amax > 0 else np.float32(1.0)\n    return fp8.e4m3_decode",
     "V scale not rounded to a power of two"),
    ("rowq-not-pow2", "oracle/dit_fp8.py",
     "s = np.where(amax > 0, pow2_ceil((amax / E4M3_MAX).astype(np.float32)), np.float32(1.0)).astype(np.float32)",
     "s = np.where(amax > 0, (amax / E4M3_MAX).astype(np.float32), np.float32(1.0)).astype(np.float32)",
     "per-row FP8 scale not rounded to a power of two"),
    ("temb-silu-dropped", "oracle/dit.py",
     'e = silu(s @ P["temb1_w"] + P["temb1_b"]) @ P["temb2_w"] + P["temb2_b"]',
     'e = (s @ P["temb1_w"] + P["temb1_b"]) @ P["temb2_w"] + P["temb2_b"]', "time MLP without its SiLU"),
    ("temb-silu-outside", "oracle/dit.py",
     'e = silu(s @ P["temb1_w"] + P["temb1_b"]) @ P["temb2_w"] + P["temb2_b"]',
     'e = silu((s @ P["temb1_w"] + P["temb1_b"]) @ P["temb2_w"] + P["temb2_b"])', "SiLU after W_e2"),
    ("temb-t-not-1000sigma", "oracle/dit.py", "s = sinusoid(1000.0 * sigma", "s = sinusoid(sigma",
     "t = sigma instead of 1000 sigma"),
    ("temb-e6-reshape-T", "oracle/dit.py", '.reshape(6, cfg.d)', '.reshape(cfg.d, 6).T', "e6 as [d,6]"),
    ("temb-e6-no-silu", "oracle/dit.py", '(silu(e) @ P["tmod_w"]', '(e @ P["tmod_w"]', "W_m on e, not SiLU(e)"),
    ("sinusoid-sin-cos", "oracle/dit.py", "np.concatenate([np.cos(t * w), np.sin(t * w)])",
     "np.concatenate([np.sin(t * w), np.cos(t * w)])", "[sin | cos] order"),
    ("txt-gelu-outside", "oracle/dit.py",
     'return gelu_tanh(ctx @ P["txt1_w"] + P["txt1_b"]) @ P["txt2_w"] + P["txt2_b"]',
     'return gelu_tanh((ctx @ P["txt1_w"] + P["txt1_b"]) @ P["txt2_w"] + P["txt2_b"])', "GELU after W_t2"),
    ("txt-b1-outside-gelu", "oracle/dit.py",
     'return gelu_tanh(ctx @ P["txt1_w"] + P["txt1_b"]) @ P["txt2_w"] + P["txt2_b"]',
     'return gelu_tanh(ctx @ P["txt1_w"]) @ P["txt2_w"] + P["txt1_b"] + P["txt2_b"]', "b_t1 outside the GELU"),
    ("ckv-k-unnormed", "oracle/dit.py",
     'k = head_rms_norm(ctxp @ P.layer(l, "ck_w") + P.layer(l, "ck_b"), cfg.heads, cfg.eps) * P.layer(l, "g_ck")',
     'k = (ctxp @ P.layer(l, "ck_w") + P.layer(l, "ck_b")) * P.layer(l, "g_ck")', "no K norm"),
    ("ckv-k-rownorm", "oracle/dit.py",
     'k = head_rms_norm(ctxp @ P.layer(l, "ck_w") + P.layer(l, "ck_b"), cfg.heads, cfg.eps) * P.layer(l, "g_ck")',
     'k = rms_norm(ctxp @ P.layer(l, "ck_w") + P.layer(l, "ck_b"), cfg.eps) * P.layer(l, "g_ck")',
     "K normalised over the whole row, not per head"),
    ("ckv-k-no-gain", "oracle/dit.py",
     'k = head_rms_norm(ctxp @ P.layer(l, "ck_w") + P.layer(l, "ck_b"), cfg.heads, cfg.eps) * P.layer(l, "g_ck")',
     'k = head_rms_norm(ctxp @ P.layer(l, "ck_w") + P.layer(l, "ck_b"), cfg.heads, cfg.eps)', "K gain dropped"),
    ("ckv-v-normed", "oracle/dit.py", 'v = ctxp @ P.layer(l, "cv_w") + P.layer(l, "cv_b")',
     'v = head_rms_norm(ctxp @ P.layer(l, "cv_w") + P.layer(l, "cv_b"), cfg.heads, cfg.eps)', "norm on V"),
    ("mod-rows-01-swapped", "oracle/dit.py", 'sh1, sc1, g1, sh2, sc2, g2 = (e6 + P.layer(l, "mod"))',
     'sc1, sh1, g1, sh2, sc2, g2 = (e6 + P.layer(l, "mod"))', "shift1/scale1 swapped"),
    ("mod-rows-34-swapped", "oracle/dit.py", 'sh1, sc1, g1, sh2, sc2, g2 = (e6 + P.layer(l, "mod"))',
     'sh1, sc1, g1, sc2, sh2, g2 = (e6 + P.layer(l, "mod"))', "shift2/scale2 swapped"),
    ("mod-gates-swapped", "oracle/dit.py", 'sh1, sc1, g1, sh2, sc2, g2 = (e6 + P.layer(l, "mod"))',
     'sh1, sc1, g2, sh2, sc2, g1 = (e6 + P.layer(l, "mod"))', "gate1/gate2 swapped"),
    ("mod-no-e6", "oracle/dit.py", 'sh1, sc1, g1, sh2, sc2, g2 = (e6 + P.layer(l, "mod"))',
     'sh1, sc1, g1, sh2, sc2, g2 = (P.layer(l, "mod"))', "M_l without e6"),
    ("mod-no-table", "oracle/dit.py", 'sh1, sc1, g1, sh2, sc2, g2 = (e6 + P.layer(l, "mod"))',
     'sh1, sc1, g1, sh2, sc2, g2 = (e6 + 0 * P.layer(l, "mod"))', "e6 without M_l"),
    ("mod1-sc-not-1+sc", "oracle/dit.py", "h = rms_norm(r, eps) * (1.0 + sc1) + sh1",
     "h = rms_norm(r, eps) * sc1 + sh1", "scale instead of 1 + scale"),
    ("mod2-swapped-inline", "oracle/dit.py", "h2 = act(rms_norm(r, eps) * (1.0 + sc2) + sh2)",
     "h2 = act(rms_norm(r, eps) * (1.0 + sh2) + sc2)", "MLP modulation with shift/scale exchanged"),
    ("swiglu-silu-on-w3", "oracle/dit.py",
     'a = silu(h2 @ wgt(l, "w1") + P.layer(l, "b1")) * (h2 @ wgt(l, "w3") + P.layer(l, "b3"))',
     'a = (h2 @ wgt(l, "w1") + P.layer(l, "b1")) * silu(h2 @ wgt(l, "w3") + P.layer(l, "b3"))',
     "SiLU on the W3 branch"),
    ("swiglu-no-b3", "oracle/dit.py",
     'a = silu(h2 @ wgt(l, "w1") + P.layer(l, "b1")) * (h2 @ wgt(l, "w3") + P.layer(l, "b3"))',
     'a = silu(h2 @ wgt(l, "w1") + P.layer(l, "b1")) * (h2 @ wgt(l, "w3"))', "b3 dropped"),
    ("mlp-bias-ungated", "oracle/dit.py", 'r = r + g2 * (act(a) @ wgt(l, "w2") + P.layer(l, "b2"))',
     'r = r + g2 * (act(a) @ wgt(l, "w2")) + P.layer(l, "b2")', "b2 outside the gate"),
    ("attn-bias-ungated", "oracle/dit.py", 'r = r + g1 * (act(_unheads(o)) @ wgt(l, "o_w") + P.layer(l, "o_b"))',
     'r = r + g1 * (act(_unheads(o)) @ wgt(l, "o_w")) + P.layer(l, "o_b")', "o_b outside the gate"),
    ("cross-gated", "oracle/dit.py", 'r = r + (act(_unheads(oc)) @ wgt(l, "co_w") + P.layer(l, "co_b"))',
     'r = r + g1 * (act(_unheads(oc)) @ wgt(l, "co_w") + P.layer(l, "co_b"))', "cross-attention gated by g1"),
    ("cross-modulated", "oracle/dit.py", 'hc = rms_norm(r, eps) * P.layer(l, "g_n3")',
     'hc = (rms_norm(r, eps) * (1.0 + sc1) + sh1) * P.layer(l, "g_n3")', "cross pre-norm modulated"),
    ("cross-no-gain", "oracle/dit.py", 'hc = rms_norm(r, eps) * P.layer(l, "g_n3")',
     'hc = rms_norm(r, eps)', "cross pre-norm gain dropped"),
    ("head-swap", "oracle/dit.py", 'sh, sc = P["head_mod"] + e', 'sc, sh = P["head_mod"] + e',
     "head shift/scale swapped"),
    ("head-no-e", "oracle/dit.py", 'sh, sc = P["head_mod"] + e', 'sh, sc = P["head_mod"] + 0 * e',
     "head ignores e"),
    ("head-sc-not-1+sc", "oracle/dit.py", 'y = (rms_norm(r, cfg.eps) * (1.0 + sc) + sh) @ P["head_w"] + P["head_b"]',
     'y = (rms_norm(r, cfg.eps) * sc + sh) @ P["head_w"] + P["head_b"]', "head: scale instead of 1 + scale"),
    ("velocity-e6-to-head", "oracle/dit.py", 'return head(P, cfg, r, cond["e"][i])',
     'return head(P, cfg, r, cond["e6"][i][0])', "head conditioned on e6 instead of e"),
    ("patch-bias-dropped", "oracle/dit.py", 'r = patchify(xin, cfg) @ P["patch_w"] + P["patch_b"]',
     'r = patchify(xin, cfg) @ P["patch_w"]', "patch-embedding bias dropped"),
    ("enc-silu-on-w3", "oracle/stages.py",
     'z = z + (dit.silu(a @ P["E.e_w1"]) * (a @ P["E.e_w3"])) @ P["E.e_w2"]',
     'z = z + ((a @ P["E.e_w1"]) * dit.silu(a @ P["E.e_w3"])) @ P["E.e_w2"]', "encoder SiLU on W3"),
    ("enc-no-residual", "oracle/stages.py",
     'z = z + (dit.silu(a @ P["E.e_w1"]) * (a @ P["E.e_w3"])) @ P["E.e_w2"]',
     'z = (dit.silu(a @ P["E.e_w1"]) * (a @ P["E.e_w3"])) @ P["E.e_w2"]', "encoder residual dropped"),
    ("enc-gains-swapped", "oracle/stages.py", 'a = dit.rms_norm(z, eps) * P["E.g_a"]',
     'a = dit.rms_norm(z, eps) * P["E.g_f"]', "encoder pre-norm uses g_f"),
    ("rope-sign", "oracle/dit.py", "out[..., 0::2] = ue * c - uo * s", "out[..., 0::2] = ue * c + uo * s",
     "RoPE rotation sign"),
    ("attn-no-scale", "oracle/dit.py", 's = np.einsum("hqd,hkd->hqk", q, k) / math.sqrt(dh)',
     's = np.einsum("hqd,hkd->hqk", q, k)', "attention without 1/sqrt(dh)"),
    ("rms-no-eps", "oracle/dit.py", "return z / np.sqrt(np.mean(z * z, axis=-1, keepdims=True) + eps)",
     "return z / np.sqrt(np.mean(z * z, axis=-1, keepdims=True) + 1e-2)", "RMSNorm eps misread (1e-2)"),
    ("euler-sign", "oracle/dit.py", "return x + (sig_next - sig_i) * v", "return x + (sig_i - sig_next) * v",
     "Euler step sign"),
]


def _run(mut, keep_going=False):
    mid, rel, old, new, what = mut
    with tempfile.TemporaryDirectory(prefix="dfmut_") as td:
        for d in ("oracle", "synth"):
            shutil.copytree(os.path.join(ROOT, d), os.path.join(td, d),
                            ignore=shutil.ignore_patterns("__pycache__", "*.so", "*.o"))
        os.makedirs(os.path.join(td, "tests"))
        for t in TESTS + ["tests/conftest.py", "tests/oracle_big.py"]:
            shutil.copy(os.path.join(ROOT, t), os.path.join(td, t))
        if old is not None:
            p = os.path.join(td, rel)
            src = open(p).read()
            if old not in src:
                return mid, what, "NOT-APPLIED", ""
            open(p, "w").write(src.replace(old, new, 1))
        env = dict(os.environ, PYTHONPATH=td, PYTHONDONTWRITEBYTECODE="1")
        # the FP8 quantisers' pins live in test_oracle_fp8.py: a mutation of fp8.py / dit_fp8.py
        # runs that file only, the others skip it (the baseline runs everything)
        fp8_only = rel in ("oracle/fp8.py", "oracle/dit_fp8.py")
        tests = TESTS if old is None else [t for t in TESTS if (t.endswith("test_oracle_fp8.py") == fp8_only)]
        r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", *tests],
                           cwd=td, env=env, capture_output=True, text=True, timeout=600)
        failed = [ln.split(" ")[1] for ln in r.stdout.splitlines() if ln.startswith("FAILED")]
        status = ("killed" if r.returncode != 0 else "SURVIVED") if old is not None else \
            ("pass" if r.returncode == 0 else "BASELINE-FAILS")
        return mid, what, status, failed[0] if failed else ""


def run_all(jobs=8):
    base = _run(("baseline", None, None, None, "unmutated oracle"))
    with cf.ThreadPoolExecutor(max_workers=jobs) as ex:
        res = list(ex.map(_run, MUTATIONS))
    return [base] + res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--log", default=None)
    ap.add_argument("-j", type=int, default=8)
    a = ap.parse_args()
    res = run_all(a.j)
    lines = [f"{'mutation':26s} {'status':10s} first failing pin  # what it models"]
    for mid, what, st, first in res:
        lines.append(f"{mid:26s} {st:10s} {first}  # {what}")
    ok = res[0][2] == "pass" and all(r[2] == "killed" for r in res[1:])
    lines.append(f"\n{sum(r[2] == 'killed' for r in res[1:])}/{len(res) - 1} mutations killed; "
                 f"baseline {res[0][2]}; {'OK' if ok else 'FAIL'}")
    out = "\n".join(lines)
    print(out)
    if a.log:
        with open(a.log, "w") as f:
            f.write(out + "\n")
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
