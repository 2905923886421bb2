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


def plan(G: int, T):
    """Exhaustive Eq. 6 maximiser over all feasible allocations."""
    if G < 3:
        raise ValueError("G < 3: no feasible allocation")
    best, key = None, None
    for gE in range(1, G - 1):
        for gT in range(1, G - gE):
            for gD in range(1, G - gE - gT + 1):
                q, _ = qps((gE, gT, gD), T)
                k = (round(q, 12), -(gE + gT + gD), gT, gD)
                if key is None or k > key:
                    best, key = (gE, gT, gD), k
    return best


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
