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
        assert 1 <= ev.g[0] <= 1 and 1 <= ev.g[1] <= 3 and 1 <= ev.g[2] <= 1   # never below 1 / above capacity
        for s in range(3):
            assert 0.0 <= ev.m.u[s] <= 1.0 and ev.m.d[s] >= 0.0
    assert any(ev.action in (1, 2, 3) for ev in log)              # the controller acted
