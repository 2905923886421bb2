"""The scheduler's decision functions in libdf (host C++, no GPU) against the oracle's
Eq. 6 planner / Alg. 1 rule / change detector and the paper's worked points."""
import os
import random

import pytest

from oracle import capacity as cap

T4 = (5.46, 74.1, 9.62)   # tab:stage_time, 4-step
T1 = (5.46, 18.7, 9.62)   # 1-step


@pytest.fixture(scope="module")
def B():
    from paper_2605_25550_b200 import binding
    if not os.path.exists(binding.LIB_PATH):
        from paper_2605_25550_b200 import build
        build.build()
    return binding


def test_plan_paper_points(B):
    assert B.plan_ratio(8, T4) == (1, 6, 1)                       # P:L532 "optimal 1:6:1"
    assert B.plan_ratio(8, T1) == (2, 4, 2)                       # Eq. 6 optimum (R25)
    assert B.plan_ratio(8, T1, cur=(1, 6, 1), budget=2) == (1, 5, 2)   # P:L532 switch
    assert B.plan_ratio(16, T4) == cap.plan(16, T4)               # P:L536 scale-out point
    assert B.plan_ratio(3, T4) == (1, 1, 1)


def test_plan_matches_oracle_random(B):
    rnd = random.Random(0)
    for _ in range(300):
        G = rnd.randint(3, 16)
        T = tuple(rnd.choice([rnd.uniform(0.5, 100.0), rnd.choice([5.0, 10.0, 20.0])]) for _ in range(3))
        cur, bud = None, -1
        if rnd.random() < 0.5:
            cur = (1, max(1, G - 3), 1)
            bud = rnd.randint(0, 6)
        want = cap.plan(G, T, cur=cur, budget=bud if cur else None)
        got = B.plan_ratio(G, T, cur=cur, budget=bud)
        assert got == want, (G, T, cur, bud)


def test_reactive_matches_oracle(B):
    cfg = B.sched_cfg(G=8)
    rnd = random.Random(1)
    for _ in range(500):
        g = [rnd.randint(1, 4) for _ in range(3)]
        now = ([rnd.random() for _ in range(3)], [rnd.choice([0, 1, 3, 6, 9]) for _ in range(3)],
               [rnd.uniform(0, 5) for _ in range(3)])
        prev = None if rnd.random() < 0.2 else ([0.5] * 3, [1] * 3, [rnd.uniform(0, 5) for _ in range(3)])
        got = B.sched_react(cfg, now, prev, g)
        want = tuple(cap.reactive(now[0][s], now[1][s], now[2][s], prev[2][s] if prev else None, g[s], sum(g), 8)
                     for s in range(3))
        assert got == want


def test_reactive_spec_examples(B):
    cfg = B.sched_cfg(G=8)
    assert B.sched_react(cfg, ([0.5, 0.95, 0.5], [2, 7, 2], [0, 4.8, 0]), ([0, 0, 0], [0, 0, 0], [0, 3.1, 0]),
                         [1, 5, 1])[1] == 1                        # ScaleOut(T)
    assert B.sched_react(cfg, ([0.5, 0.5, 0.1], [2, 2, 0], [0, 0, 0]), None, [1, 5, 2])[2] == -1  # ScaleIn(D)
    assert B.sched_react(cfg, ([0.5, 0.5, 0.5], [2, 2, 2], [1, 1, 1]), None, [1, 5, 2]) == (0, 0, 0)


def test_change_detector_matches_oracle(B):
    rnd = random.Random(2)
    for _ in range(300):
        n = rnd.randint(0, 40)
        keys = [rnd.choice([1, 4, 8, 28]) for _ in range(n)]
        if rnd.random() < 0.5 and n > 8:
            keys = [4] * (n - n // 4) + [1] * (n // 4)
        assert B.sched_changed(keys) == cap.changed(keys), keys


def _tile_check(pieces, total):
    """Every byte of [0, total) is covered by exactly one piece."""
    import numpy as np
    cover = np.zeros(total, np.int32)
    for off, width, height, pitch in pieces:
        for r in range(height):
            cover[off + r * pitch: off + r * pitch + width] += 1
    return bool(np.all(cover == 1))


@pytest.mark.parametrize("cfg_name,chunks", [("tiny", (64, 256)), ("mid", (4096, 16384)), ("image", (524288, 131072)),
                                             ("video", (524288, 131072)), ("image", (0, 0)), ("mid", (1000, 3000))])
def test_chunk_plans_tile_the_payloads(B, cfg_name, chunks):
    """R22 host logic (no GPU): the E->T plan cuts the ctx payload into whole rows, the T->D plan
    cuts the latent into per-frame row blocks (one frame per chunk for video, 16 latent rows at
    the image shape with 128 KiB), and both tile their payload exactly once."""
    from synth.configs import CONFIGS
    cfg = CONFIGS[cfg_name]
    g = B.make_graph(cfg, [(0, B.DF_E), (0, B.DF_T), (0, B.DF_D)], chunk_bytes=chunks)
    ctx_bytes = cfg.L_txt * cfg.d_txt * 2
    p0 = B.chunk_plan(g, 0, ctx_bytes)
    assert _tile_check(p0, ctx_bytes)
    row = cfg.d_txt * 2
    assert all(w % row == 0 or off + w == ctx_bytes for off, w, h, pt in p0)   # whole rows
    lat = cfg.C * cfg.F * cfg.H * cfg.W * 4
    p1 = B.chunk_plan(g, 1, lat)
    assert _tile_check(p1, lat)
    if chunks[1] == 0:
        assert len(p1) == 1
    elif cfg.F > 1:
        assert len(p1) == cfg.F and all(h == cfg.C for _, _, h, _ in p1)    # one latent frame each
    elif cfg_name == "image":
        assert len(p1) == 8 and p1[0][1] == 16 * cfg.W * 4                  # 16-row blocks
