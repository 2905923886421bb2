"""ORACLE (test infrastructure only — see oracle/__init__.py).

Closed forms of the paper's instance-scheduling model and of the stage handoff.

* Eq. 1: g_E + g_T + g_D <= G.
* Eq. 6: QPS = min{g_E/T_E, g_T/T_T, g_D/T_D}.
* Eq. 7: the optimum balances the per-stage rates; the planner
  is the exhaustive maximiser of Eq. 6 (SPEC S:L527 reading; ties: fewer GPUs,
  then larger g_T, then larger g_D).
* The tensor-hash check: the downstream stage verifies the received
  tensor equals what upstream sent.  The hash is DESIGN.md's definition:
  H(bytes) = sum_i splitmix64(w_i XOR (i * 0x9E3779B97F4A7C15)) mod 2^64 over the
  little-endian uint64 words w_i of the zero-padded payload.
* Jitter ("p% chance of +d s"): one Bernoulli draw per request-edge
  transfer (R23): delayed iff Philox(seed; req, edge) word < p * 2^32.
"""
from __future__ import annotations

import numpy as np

from .philox import philox4x32_10

GOLDEN = 0x9E3779B97F4A7C15
U64 = np.uint64


def qps(g, T):
    """Eq. 6. g = (gE, gT, gD), T = (T_E, T_T, T_D) seconds -> (req/s, bottleneck stage)."""
    rates = [g[s] / T[s] for s in range(3)]
    b = int(np.argmin(rates))  # ties E < T < D
    return rates[b], "ETD"[b]


def feasible(g, G) -> bool:
    """Eq. 1 plus one instance per stage."""
    return min(g) >= 1 and sum(g) <= G


def plan(G: int, T, cur=None, budget=None):
    """Exhaustive Eq. 6 maximiser over all feasible allocations; with `cur` and `budget`,
    only allocations within `budget` instance moves (L1 distance) of `cur`."""
    if G < 3:
        raise ValueError("G < 3: no feasible allocation")
    best, key = None, None
    for gE in range(1, G - 1):
        for gT in range(1, G - gE):
            for gD in range(1, G - gE - gT + 1):
                if cur is not None and budget is not None and budget >= 0 and \
                        abs(gE - cur[0]) + abs(gT - cur[1]) + abs(gD - cur[2]) > budget:
                    continue
                q, _ = qps((gE, gT, gD), T)
                k = (round(q, 12), -(gE + gT + gD), gT, gD)
                if key is None or k > key:
                    best, key = (gE, gT, gD), k
    return best


def reactive(u, q, d, d_prev, g_s, g_total, G, U_high=0.8, Q_high=5, U_low=0.2):
    """Alg. 1 lines 11-17 for one service s with g_s instances: +1 (ScaleOut)
    iff u > U_high and q > Q_high and d > d' (previous window; the first tick has none)
    and a GPU is free (g_total < G, Eq. 1); -1 (ScaleIn) iff u < U_low and q = 0, never
    below one instance; else 0."""
    if u > U_high and q > Q_high and d_prev is not None and d > d_prev:
        return 1 if g_total < G else 0
    if u < U_low and q == 0:
        return -1 if g_s >= 2 else 0
    return 0


def changed(keys) -> bool:
    """Changed(H) (Alg. 1 line 6; "identifying the most frequent workload in H"):
    the modal key of the most recent 25% differs from the modal key of the rest; a tie
    for the mode in either part means no change (SPEC S:L490 reading)."""
    n = len(keys)
    if n < 4:
        return False
    cut = n - max(1, n // 4)

    def mode(xs):
        from collections import Counter
        c = Counter(xs).most_common()
        if len(c) > 1 and c[0][1] == c[1][1]:
            return None
        return c[0][0]
    a, b = mode(keys[:cut]), mode(keys[cut:])
    return a is not None and b is not None and a != b


def splitmix64(z: np.ndarray) -> np.ndarray:
    z = np.asarray(z, dtype=U64)
    with np.errstate(over="ignore"):
        z = z + U64(GOLDEN)
        z = (z ^ (z >> U64(30))) * U64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> U64(27))) * U64(0x94D049BB133111EB)
        return z ^ (z >> U64(31))


def payload_hash(buf: bytes | np.ndarray, word_offset: int = 0) -> int:
    """DESIGN.md payload hash; word_offset lets a chunk starting at byte 8*o be
    hashed alone (the total is the mod-2^64 sum of the chunks' hashes)."""
    b = np.frombuffer(bytes(buf), dtype=np.uint8) if not isinstance(buf, np.ndarray) else buf.view(np.uint8).reshape(-1)
    pad = (-b.size) % 8
    if pad:
        b = np.concatenate([b, np.zeros(pad, dtype=np.uint8)])
    w = b.view("<u8").astype(U64)
    idx = np.arange(word_offset, word_offset + w.size, dtype=U64)
    with np.errstate(over="ignore"):
        h = splitmix64(w ^ (idx * U64(GOLDEN)))
        return int(np.sum(h, dtype=U64))


def chunks(nbytes: int, chunk: int):
    """[(offset, size)] of the chunked handoff; chunk 0 = whole payload."""
    if chunk <= 0 or chunk >= nbytes:
        return [(0, nbytes)] if nbytes else []
    return [(o, min(chunk, nbytes - o)) for o in range(0, nbytes, chunk)]


def jitter_delayed(seed: int, req: int, edge: int, p: float) -> bool:
    w = philox4x32_10(np.array([req & 0xFFFFFFFF], U64), np.array([req >> 32], U64),
                      np.array([edge], U64), np.array([3], U64),
                      seed & 0xFFFFFFFF, seed >> 32)[0][0]
    return int(w) < int(p * 4294967296.0)
