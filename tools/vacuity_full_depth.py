"""Vacuity guard of the fp64 oracle at the C2 / C3 widths AND depths on a
reduced token grid (one latent frame of 16x16 -> N = 64 tokens; full d, heads, f, L_txt,
layers).  Test infrastructure: calls only oracle/ and synth/.

    python tools/vacuity_full_depth.py image|video [--out profiles/r02_vacuity_<cfg>.json]

Reports per block rho_l = ||r_{l+1} - r_l|| / ||r_l|| (must lie in [1e-2, 1]), ||v||/||x||
(in [0.1, 10]) and the relative change of v when cross-attention is removed (>= 5e-2)."""
import argparse
import dataclasses
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from synth.configs import CONFIGS  # noqa: E402
from synth import inputs  # noqa: E402
from oracle import params as OP, dit  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--layers", type=int, default=0)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    base = CONFIGS[a.config]
    cfg = dataclasses.replace(base, F=1, H=16, W=16, layers=a.layers or base.layers)
    t0 = time.time()
    P = OP.Params(cfg, 0)
    sig = dit.sigmas(cfg.steps, cfg.shift)
    ctx = inputs.bf16_bits_to_f64(inputs.ctx_bf16(cfg, 0))
    # dit.velocity's composition, evaluated layer by layer so that only one layer's weights
    # are resident (C3 at fp64 is 135 GB): patch embed -> blocks -> head, step i = 1, with
    # and without cross-attention in the same pass
    ctxp = dit.text_projection(P, cfg, ctx)
    e, e6 = dit.time_embedding(P, cfg, float(sig[1]))
    pos = dit.token_positions(cfg)
    x = inputs.latent(cfg, 0).astype(np.float64)
    r = dit.patchify(x, cfg) @ P["patch_w"] + P["patch_b"]
    r0 = r.copy()
    rho = []
    for l in range(cfg.layers):
        kv = dit.cross_kv(P, cfg, l, ctxp)
        rn = dit.block(P, cfg, l, r, e6, kv, pos)
        rho.append(float(np.linalg.norm(rn - r) / np.linalg.norm(r)))
        r = rn
        r0 = dit.block(P, cfg, l, r0, e6, kv, pos, cross=False)
        for k in [k for k in P._cache if k.startswith(f"L{l}.")]:
            del P._cache[k]
        print(f"layer {l}: rho {rho[-1]:.4f} ({time.time() - t0:.0f} s)", file=sys.stderr, flush=True)
    v = dit.head(P, cfg, r, e)
    v0 = dit.head(P, cfg, r0, e)
    res = {"config": a.config, "N": cfg.N, "d": cfg.d, "layers": cfg.layers, "step": 1, "rho": rho,
           "rho_min": min(rho), "rho_max": max(rho), "v_over_x": float(np.linalg.norm(v) / np.linalg.norm(x)),
           "cross_effect": float(np.linalg.norm(v - v0) / np.linalg.norm(v)), "seconds": time.time() - t0}
    res["pass"] = (all(1e-2 <= r <= 1.0 for r in rho) and 0.1 <= res["v_over_x"] <= 10.0
                   and res["cross_effect"] >= 5e-2)
    print(json.dumps(res))
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
