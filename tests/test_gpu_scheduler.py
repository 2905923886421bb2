"""The Alg. 1 controller on a live pipeline: it measures u/q/d per stage, detects the
4-step -> 1-step workload switch (the paper's §5.6 parameter trace) and
reconfigures through df_set_ratio without losing a request."""
import time

import numpy as np
import pytest

from synth.configs import TINY
from gpu_util import make_ctx

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
from paper_2605_25550_b200 import binding as B  # noqa: E402


def test_controller_reacts_to_workload_switch():
    inst = [(0, B.DF_E), (0, B.DF_T), (0, B.DF_T), (0, B.DF_T), (0, B.DF_D)]
    with make_ctx(TINY, instances=inst) as c:
        c.sched_start(B.sched_cfg(delta_s=0.1, G=5))
        seeds = list(range(200))
        comps = []
        for k, s in enumerate(seeds):
            steps = 4 if k < 100 else 1
            while c.submit(steps, TINY.shift, s, user_tag=s)[0] != B.DF_OK:
                comps += c.poll(32, 5)
            if k % 20 == 19:
                time.sleep(0.15)  # let the controller tick inside each regime
        while len(comps) < len(seeds):
            comps += c.poll(64, 10000)
        time.sleep(0.3)
        c.sched_stop()
        log = c.sched_log()
    assert sorted(x.user_tag for x in comps) == seeds             # conservation, no loss
    assert len(log) >= 3
    for ev in log:
        assert min(ev.g) >= 1 and sum(ev.g) <= 5                  # never below 1 / above the 5 hosts
        if ev.action != 4:
            for s in range(3):
                assert 0.0 <= ev.m.u[s] <= 1.0 and ev.m.d[s] >= 0.0
    assert any(ev.action in (1, 2, 3) for ev in log)              # the controller acted


def _run(c, cfg, seeds, steps=3):
    outs = {s: np.zeros(cfg.out_shape, np.float32) for s in seeds}
    for s in seeds:
        while c.submit(steps, 3.0, s, out_host=outs[s], user_tag=s)[0] != B.DF_OK:
            time.sleep(0.001)
    comps = []
    while len(comps) < len(seeds):
        comps += c.poll(16, timeout_ms=60000)
    return outs, comps


def test_set_ratio_repurposes_an_instance_with_a_cold_start():
    """Alg. 1 "Apply" with re-purposing ("cold starts and reclamation"): hosts
    [E, E, T, D] on one GPU.  set_ratio(1, 2, 1) has one T too few, so the surplus E (instance 1)
    is drained, freed and re-created as a DiT instance (weights regenerated from the seed: the
    measured cold start) and serves; set_ratio(2, 1, 1) moves it back.  No request is lost, and
    every request's output bytes equal those of a context that never re-purposed (P15)."""
    from synth.configs import MID
    cfg = MID
    inst = [(0, B.DF_E), (0, B.DF_E), (0, B.DF_T), (0, B.DF_D)]
    with make_ctx(cfg, instances=inst, chunk_bytes=(4096, 16384)) as c:
        o1, c1 = _run(c, cfg, [1, 2, 3])
        assert c.set_ratio(1, 2, 1) == B.DF_OK
        ev = [e for e in c.sched_log() if e.action == 4]
        assert len(ev) == 1 and ev[0].inst == 1 and ev[0].from_stage == B.DF_E and ev[0].stage == B.DF_T
        assert ev[0].cold_start_ms > 0 and ev[0].drain_ms >= 0
        o2, c2 = _run(c, cfg, list(range(10, 18)))
        assert {x.inst[1] for x in c2} == {1, 2}                  # the new DiT instance serves
        assert c.set_ratio(2, 1, 1) == B.DF_OK                     # and goes back to encoding
        ev = [e for e in c.sched_log() if e.action == 4]
        assert len(ev) == 2 and ev[1].inst == 1 and ev[1].from_stage == B.DF_T and ev[1].stage == B.DF_E
        o3, c3 = _run(c, cfg, list(range(20, 26)))
        assert {x.inst[0] for x in c3} <= {0, 1} and {x.inst[1] for x in c3} == {2}
        assert c.set_ratio(1, 3, 1) == B.DF_ERR_CAPACITY           # 5 > 4 hosts (Eq. 1)
    for comps, seeds in ((c1, [1, 2, 3]), (c2, list(range(10, 18))), (c3, list(range(20, 26)))):
        assert sorted(x.user_tag for x in comps) == seeds
        assert all(x.hash_src[e] == x.hash_dst[e] != 0 for x in comps for e in range(2))
    with make_ctx(cfg, chunk_bytes=(4096, 16384)) as c:
        ref, _ = _run(c, cfg, [2, 11, 12, 21])
    for s, o in ((2, o1), (11, o2), (12, o2), (21, o3)):
        assert np.array_equal(o[s], ref[s]), s
