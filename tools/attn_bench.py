"""Attention microbenchmark through df_op_attention (no model): TFLOP/s of the tcgen05
flash-attention kernel at the workload shapes.  DF_ATTN_IMPL=2 (read once per process)
selects the attn_tc2 A/B kernel instead of the default persistent attn_pp at dh = 128.

    python tools/attn_bench.py --shape video
"""
import argparse
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_25550_b200 import binding as B  # noqa: E402
from synth.configs import TINY  # noqa: E402

SHAPES = {"video": (40, 32760, 32760), "image": (24, 4096, 4096), "cross_video": (40, 32760, 512),
          "cross_image": (24, 4096, 512)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="video")
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--lib", action="store_true", help="also time torch SDPA (cuDNN / flash backends) on the same inputs")
    ap.add_argument("--H", type=int, default=0, help="override the head count (work-item scaling experiments)")
    ap.add_argument("--reps", type=int, default=1, help="back-to-back launches per timed sample (amortises launch latency)")
    ap.add_argument("--f8", type=int, default=0, help="1: e4m3 Q/K (R32); 2: e4m3 Q/K/V and P (R33) -- FP8 modes")
    a = ap.parse_args()
    H, Nq, Nk = SHAPES[a.shape]
    if a.H:
        H = a.H
    dh = 128
    g = B.make_graph(TINY, [(0, B.DF_E), (0, B.DF_T), (0, B.DF_D)])
    with B.Context(g) as c:
        torch.manual_seed(0)

        def rmsn(t):  # RMS-normalised rows like the model's qk-norm (R6)
            return t * torch.rsqrt(t.float().pow(2).mean(-1, keepdim=True)).to(t.dtype)
        Q = rmsn(torch.randn(H, Nq, dh, device="cuda")).to(torch.bfloat16)
        K = rmsn(torch.randn(H, Nk, dh, device="cuda")).to(torch.bfloat16)
        V = torch.randn(H, Nk, dh, device="cuda").to(torch.bfloat16)
        O = torch.empty(Nq, H * dh, device="cuda", dtype=torch.bfloat16)
        sc = 1.0 / math.sqrt(dh)
        run = lambda: c.op_attention(Q, K, V, O, H, Nq, Nk, dh, dh, sc)  # noqa: E731
        if a.f8:  # unit gains: s = pow2ceil(sqrt(128) / 448) = 2^-5 for Q and K
            s8 = 2.0 ** -5
            Q8 = torch.empty((H, Nq, dh), dtype=torch.uint8, device="cuda")
            K8 = torch.empty((H, Nk, dh), dtype=torch.uint8, device="cuda")
            c.op_qk_e4m3(Q, 1.0 / s8, Q8)
            c.op_qk_e4m3(K, 1.0 / s8, K8)
            if a.f8 == 1:
                run = lambda: c.op_attention_qf8(Q8, K8, V, O, H, Nq, Nk, sc * s8 * s8)  # noqa: E731
            else:
                v8t = torch.zeros((H, 128, (Nk + 63) // 64 * 64), dtype=torch.uint8, device="cuda")
                vs = torch.zeros(2, device="cuda")
                run = lambda: c.op_attention_f8(Q8, K8, V, O, H, Nq, Nk, sc * s8 * s8, v8t, vs)  # noqa: E731
        run()
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ms = []
        for _ in range(a.iters):
            ev[0].record()
            for _ in range(a.reps):
                run()
            ev[1].record()
            torch.cuda.synchronize()
            ms.append(ev[0].elapsed_time(ev[1]) / a.reps)
        rows = torch.arange(0, Nq, max(1, Nq // 7), device="cuda")[:8]
        qf, kf, vf = Q[:, rows].float(), K.float(), V.float()
        ref = torch.softmax(qf @ kf.transpose(1, 2) * sc, -1) @ vf
        got = O[rows].float().view(len(rows), H, dh).transpose(0, 1)
        err = ((got - ref).norm() / ref.norm()).item()
        fl = 4.0 * H * Nq * Nk * dh
        best = min(ms)
        print({"shape": a.shape, "H": H, "impl": os.environ.get("DF_ATTN_IMPL", "default"), "f8": a.f8,
               "ms": round(best, 3), "tflops": round(fl / best / 1e9, 1),
               "rel_l2_vs_torch": f"{err:.2e}"})
        if a.lib:  # library reference point (not on the product path)
            from torch.nn.attention import SDPBackend, sdpa_kernel
            q4, k4, v4 = Q.unsqueeze(0), K.unsqueeze(0), V.unsqueeze(0)
            for be in (SDPBackend.CUDNN_ATTENTION, SDPBackend.FLASH_ATTENTION):
                try:
                    with sdpa_kernel(be):
                        f = lambda: torch.nn.functional.scaled_dot_product_attention(q4, k4, v4, scale=sc)
                        f()
                        torch.cuda.synchronize()
                        lm = []
                        for _ in range(a.iters):
                            ev[0].record()
                            for _ in range(a.reps):
                                f()
                            ev[1].record()
                            torch.cuda.synchronize()
                            lm.append(ev[0].elapsed_time(ev[1]) / a.reps)
                    print({"shape": a.shape, "lib": str(be), "ms": round(min(lm), 3),
                           "tflops": round(fl / min(lm) / 1e9, 1)}, flush=True)
                except Exception as ex:  # backend not available for this shape / build
                    print({"shape": a.shape, "lib": str(be), "error": str(ex)[:120]}, flush=True)


if __name__ == "__main__":
    main()
