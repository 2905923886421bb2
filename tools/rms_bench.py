"""RMSNorm+modulation microbenchmark (df_op_rmsnorm_mod): achieved GB/s (fp32 read + bf16
write) at the image and video row shapes, back-to-back launches vs a single launch.

    python tools/rms_bench.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_25550_b200 import binding as B  # noqa: E402
from synth.configs import TINY  # noqa: E402


def main():
    g = B.make_graph(TINY, [(0, B.DF_E), (0, B.DF_T), (0, B.DF_D)])
    with B.Context(g) as c:
        for M, d in ((4096, 3072), (8192, 3072), (32760, 5120)):
            x = torch.randn(M, d, device="cuda")
            sh = torch.randn(d, device="cuda") * 0.1
            sc = torch.randn(d, device="cuda") * 0.1
            out = torch.empty(M, d, device="cuda", dtype=torch.bfloat16)
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            for reps in (1, 20):
                c.op_rmsnorm_mod(x, out, sh, sc, 1e-6)
                torch.cuda.synchronize()
                ev[0].record()
                for _ in range(reps):
                    c.op_rmsnorm_mod(x, out, sh, sc, 1e-6)
                ev[1].record()
                torch.cuda.synchronize()
                us = ev[0].elapsed_time(ev[1]) * 1e3 / reps
                print({"M": M, "d": d, "reps": reps, "us": round(us, 2),
                       "GB/s": round(M * d * 6 / us / 1e3, 1)}, flush=True)


if __name__ == "__main__":
    main()
