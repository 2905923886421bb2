"""GEMM microbenchmark: libdf's tcgen05 CTA-pair GEMM (df_op_gemm, fp32 output) against
cuBLAS bf16 (torch.matmul, bf16 output) on the same shapes, same run — separates the
mainloop from the fused epilogues measured inside the DiT step.

    python tools/gemm_bench.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_25550_b200 import binding as B  # noqa: E402
from synth.configs import TINY  # noqa: E402

SHAPES = [("square8192", 8192, 8192, 8192), ("image_qkv", 4096, 9216, 3072), ("image_up", 4096, 16384, 3072),
          ("image_o", 4096, 3072, 3072), ("image_down", 4096, 3072, 8192), ("video_up", 32760, 27648, 5120)]


def timeit(fn, iters=10):
    fn()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    best = 1e30
    for _ in range(iters):
        ev[0].record()
        fn()
        ev[1].record()
        torch.cuda.synchronize()
        best = min(best, ev[0].elapsed_time(ev[1]))
    return best


def fp8_shape(c, name, A, W, M, N, K, no_cublas):
    """NEXT-4: per-tensor e4m3 operands (quantised by df_op_quant_e4m3), bf16 output."""
    qa = torch.empty(M, K, dtype=torch.uint8, device="cuda")
    qb = torch.empty(N, K, dtype=torch.uint8, device="cuda")
    sa = torch.empty(1, device="cuda")
    sb = torch.empty(1, device="cuda")
    ms_q = timeit(lambda: c.op_quant_e4m3(A, qa, sa))
    c.op_quant_e4m3(W, qb, sb)
    out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    ms_ours = timeit(lambda: c.op_gemm_e4m3(qa, qb, sa, sb, out))
    fl = 2.0 * M * N * K
    row = {"shape": name, "dtype": "e4m3", "M": M, "N": N, "K": K, "ours_tflops": round(fl / ms_ours / 1e9, 1),
           "quant_A_gbs": round(A.numel() * 3 / ms_q / 1e6, 1)}
    if not no_cublas:
        fa, fb = qa.view(torch.float8_e4m3fn), qb.view(torch.float8_e4m3fn)
        ms_lib = timeit(lambda: torch._scaled_mm(fa, fb.t(), scale_a=sa, scale_b=sb, out_dtype=torch.bfloat16))
        ref = torch._scaled_mm(fa, fb.t(), scale_a=sa, scale_b=sb, out_dtype=torch.bfloat16).float()
        row.update({"cublaslt_tflops": round(fl / ms_lib / 1e9, 1), "ratio": round(ms_lib / ms_ours, 3),
                    "rel_err_vs_cublaslt": f"{((out.float() - ref).norm() / ref.norm()).item():.1e}"})
    print(row, flush=True)


def mx_shape(c, name, A, W, M, N, K, no_cublas):
    """NEXT-4 MXFP8 (R30): OCP MX e4m3 operands with E8M0 block-32 scales (df_op_mx_quant_e4m3),
    the block-scaled GEMM (df_op_gemm_mxf8), bf16 out; the per-tensor e4m3 GEMM on the same
    shape for comparison."""
    sfn = lambda R: (K // 128) * ((R + 127) // 128) * 512
    qa = torch.empty(M, K, dtype=torch.uint8, device="cuda")
    qb = torch.empty(N, K, dtype=torch.uint8, device="cuda")
    sa = torch.empty(sfn(M), dtype=torch.uint8, device="cuda")
    sb = torch.empty(sfn(N), dtype=torch.uint8, device="cuda")
    ms_q = timeit(lambda: c.op_mx_quant_e4m3(A, qa, sa))
    c.op_mx_quant_e4m3(W, qb, sb)
    out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    ms_mx = timeit(lambda: c.op_gemm_mxf8(qa, sa, qb, sb, out))
    fl = 2.0 * M * N * K
    ref = A.float() @ W.float().t()
    err = ((out.float() - ref).norm() / ref.norm()).item()
    one = torch.ones(1, device="cuda")
    out2 = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    ms_pt = timeit(lambda: c.op_gemm_e4m3(qa, qb, one, one, out2))
    print({"shape": name, "dtype": "mxf8", "M": M, "N": N, "K": K, "mx_tflops": round(fl / ms_mx / 1e9, 1),
           "e4m3_per_tensor_tflops": round(fl / ms_pt / 1e9, 1), "rel_err_vs_bf16_product": f"{err:.2e}",
           "quant_A_gbs": round(A.numel() * (3 + 1 / 32) / ms_q / 1e6, 1)}, flush=True)


def main():
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="")
    ap.add_argument("--no-cublas", action="store_true")
    ap.add_argument("--tc", type=int, default=1, help="2: allow the stream-K schedule")
    ap.add_argument("--fp8", action="store_true", help="e4m3 GEMM (df_op_gemm_e4m3) vs cuBLASLt torch._scaled_mm")
    ap.add_argument("--mx", action="store_true", help="MXFP8 block-scaled GEMM (df_op_gemm_mxf8)")
    a = ap.parse_args()
    g = B.make_graph(TINY, [(0, B.DF_E), (0, B.DF_T), (0, B.DF_D)])
    with B.Context(g) as c:
        for name, M, N, K in SHAPES:
            if a.only and name != a.only:
                continue
            A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
            W = torch.randn(N, K, device="cuda").to(torch.bfloat16)
            if a.mx:
                mx_shape(c, name, A, W, M, N, K, a.no_cublas)
                del A, W
                continue
            if a.fp8:
                fp8_shape(c, name, A, W, M, N, K, a.no_cublas)
                del A, W
                continue
            out = torch.empty(M, N, device="cuda")
            ms_ours = timeit(lambda: c.op_gemm(A, W, out, tc=a.tc))
            ms_cublas = ms_ours if a.no_cublas else timeit(lambda: torch.matmul(A, W.t()))
            fl = 2.0 * M * N * K
            ref = (A.float() @ W.float().t())
            err = ((out - ref).norm() / ref.norm()).item()
            print({"shape": name, "tc": a.tc, "M": M, "N": N, "K": K, "ours_tflops": round(fl / ms_ours / 1e9, 1),
                   "cublas_tflops": round(fl / ms_cublas / 1e9, 1), "ratio": round(ms_cublas / ms_ours, 3),
                   "rel_err": f"{err:.1e}"}, flush=True)
            del A, W, out, ref


if __name__ == "__main__":
    main()
