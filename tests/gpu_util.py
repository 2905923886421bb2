"""Helpers shared by the -m gpu parity tests (test code only)."""
import numpy as np


def rel_l2(a, b) -> float:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def bf16_tensor_from_bits(bits, device="cuda"):
    import torch
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).to(device).view(torch.bfloat16)


def bf16_bits_of(t):
    import torch
    return t.detach().contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def make_ctx(cfg, precision=0, seed=0, instances=None, **kw):
    from paper_2605_25550_b200 import binding as B
    inst = instances or [(0, B.DF_E), (0, B.DF_T), (0, B.DF_D)]
    return B.Context(B.make_graph(cfg, inst, precision=precision, weight_seed=seed, **kw))
