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
