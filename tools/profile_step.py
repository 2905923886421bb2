"""Drive a short, ncu-friendly slice of the hot path: prologue + `--steps` DiT steps
(first step = warm-up) of one request at a BASELINE workload shape, through the C ABI.

    ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file launches.csv \
        python tools/profile_step.py --config image --steps 2
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_25550_b200 import binding as B  # noqa: E402
from synth.configs import CONFIGS, with_layers  # noqa: E402
from synth import inputs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="image")
    ap.add_argument("--layers", type=int, default=0)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--kstats", action="store_true")
    ap.add_argument("--precision", default="bf16", choices=["bf16", "fp8", "mxfp8"])
    a = ap.parse_args()
    cfg = CONFIGS[a.config]
    if a.layers:
        cfg = with_layers(cfg, a.layers)
    prec = {"fp8": B.DF_FP8, "mxfp8": B.DF_MXFP8}.get(a.precision, B.DF_BF16)
    g = B.make_graph(cfg, [(0, B.DF_E), (0, B.DF_T), (0, B.DF_D)], max_steps=cfg.steps, precision=prec)
    with B.Context(g) as c:
        ctx = torch.from_numpy(inputs.ctx_bf16(cfg, 1).view(np.int16)).cuda().view(torch.bfloat16)
        s = np.linspace(1, 0, cfg.steps + 1).astype(np.float32)
        cond = c.dit_prepare(1, ctx, s)
        if a.kstats:
            c.profile(True, True)
        x = torch.from_numpy(inputs.latent(cfg, 2)).cuda()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps + 1)]
        ev[0].record()
        for i in range(a.steps):
            c.dit_step(1, cond, i, x)
            ev[i + 1].record()
        torch.cuda.synchronize()
        ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(a.steps)]
        fl = cfg.flops_per_step()
        print({"config": cfg.name, "layers": cfg.layers, "step_ms": ms,
               "tflops": [fl / (m / 1e3) / 1e12 for m in ms]})
        if a.kstats:
            ks = c.kernel_stats()
            tot = sum(v["ms"] for v in ks.values())
            for k, v in ks.items():
                if v["launches"]:
                    avg = v["ms"] / v["launches"]
                    print(f"  {k:12s} share {v['ms'] / tot:6.3f}  avg {avg * 1e3:8.1f} us  "
                          f"{(v['flops'] / v['ms'] / 1e9) if v['flops'] else (v['bytes'] / v['ms'] / 1e6):8.1f} "
                          f"{'TFLOP/s' if v['flops'] else 'GB/s'}")
        c.cond_release(cond)


if __name__ == "__main__":
    main()
