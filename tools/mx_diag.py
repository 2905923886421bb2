"""MXFP8 scale-factor layout diagnostic (bring-up of R30's block-scaled GEMM): decode which
scale byte the tensor core applied to each (row, k-block) by making one k-block of A nonzero
and filling the scale buffers with offset-encoding bytes."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_25550_b200 import binding as B  # noqa: E402
from synth.configs import TINY  # noqa: E402

M = N = 256
K = 128
ONE = 0x38  # e4m3 1.0


def run(c, qa, sa, qb, sb):
    out = torch.full((M, N), float("nan"), device="cuda")
    c.op_gemm_mxf8(torch.from_numpy(qa).cuda(), torch.from_numpy(sa).cuda(), torch.from_numpy(qb).cuda(),
                   torch.from_numpy(sb).cuda(), out)
    torch.cuda.synchronize()
    return out.cpu().numpy().astype(np.float64)


def expected(r, kb):
    return (r // 128) * 512 + (r % 32) * 16 + ((r % 128) // 32) * 4 + kb % 4


def main():
    g = B.make_graph(TINY, [(0, B.DF_E), (0, B.DF_T), (0, B.DF_D)])
    nbytes = (K // 128) * 2 * 512
    o = np.arange(nbytes)
    with B.Context(g) as c:
        for side in ("A", "B"):
            res = {}
            for kb in range(4):
                qa = np.zeros((M, K), np.uint8)
                qb = np.zeros((N, K), np.uint8)
                if side == "A":
                    qa[:, kb * 32:(kb + 1) * 32] = ONE
                    qb[:, :] = ONE
                else:
                    qa[:, :] = ONE
                    qb[:, kb * 32:(kb + 1) * 32] = ONE
                dec = []
                for pat in (60 + (o % 128), 60 + (o // 128)):
                    sfx = pat.astype(np.uint8)
                    ones = np.full(nbytes, 127, np.uint8)
                    out = run(c, qa, sfx if side == "A" else ones, qb, ones if side == "A" else sfx)
                    v = out[:, 0] if side == "A" else out[0, :]
                    with np.errstate(divide="ignore", invalid="ignore"):
                        e = np.log2(np.abs(v) / 32.0) + 127 - 60
                    dec.append(e)
                got = np.where(np.isfinite(dec[0]) & np.isfinite(dec[1]), np.round(dec[1]) * 128 + np.round(dec[0]), -1)
                res[kb] = got.astype(int)
            bad = 0
            for kb in range(4):
                exp = np.array([expected(r, kb) for r in range(256)])
                bad += int(np.sum(res[kb] != exp))
            print(f"side {side}: mismatches vs expected layout: {bad} of 1024")
            for kb in range(4):
                print(f"  {side} kb {kb} used:", " ".join(str(int(x)) for x in res[kb]))


if __name__ == "__main__":
    main()
