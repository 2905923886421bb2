"""Stage-partitioned layouts of the E -> T -> D pipeline over N GPUs of one node
("allocate a certain number of instances to the three
stages"; Eq. 1 g_E + g_T + g_D <= G with co-location allowed on B200 because every
stage's weights fit in 180 GB).

A layout is a list of (device, stage, rank) instances for df_graph, one process
(rank) per GPU, device = the process's local CUDA device.
"""
from __future__ import annotations

from .binding import DF_E, DF_T, DF_D


def partitioned(n_gpus: int, exclusive: bool = False, t_per_gpu: int = 1):
    """DiT instances data-parallel over requests; E on GPU 0, D on the last GPU.

    exclusive=False (default): one T instance on every GPU (E:T:D = 1:N:1, E and D
    co-located with a T) — the Eq. 6 optimum on B200 where T_E, T_D << T_T.
    t_per_gpu > 1 places several DiT instances (own weights, own streams) on each GPU: their
    persistent kernels fill the SMs left idle by each other's wave-quantisation tails.
    exclusive=True: E and D get GPUs of their own (the paper's 1:6:1 at N = 8)."""
    if n_gpus < 1 or t_per_gpu < 1:
        raise ValueError("n_gpus >= 1, t_per_gpu >= 1")
    if n_gpus == 1:
        return [(0, DF_E, 0)] + [(0, DF_T, 0)] * t_per_gpu + [(0, DF_D, 0)]
    if exclusive:
        if n_gpus < 3:
            raise ValueError("exclusive layout needs >= 3 GPUs")
        inst = [(0, DF_E, 0)] + [(0, DF_T, r) for r in range(1, n_gpus - 1) for _ in range(t_per_gpu)] + \
            [(0, DF_D, n_gpus - 1)]
    else:
        inst = [(0, DF_E, 0)] + [(0, DF_T, r) for r in range(n_gpus) for _ in range(t_per_gpu)] + \
            [(0, DF_D, n_gpus - 1)]
    return inst


def ratio(inst):
    """(g_E, g_T, g_D) of a layout."""
    return tuple(sum(1 for i in inst if i[1] == s) for s in (DF_E, DF_T, DF_D))


def ranks_of(inst, stage):
    return sorted({i[2] for i in inst if i[1] == stage})
