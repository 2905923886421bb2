"""BASELINE configs[3] "workload shift": a request stream whose DiT cost drops mid-run (the
paper's 4-step -> 1-step switch, here at the image shape: 28-step then 1-step
requests) served with the hybrid instance scheduler (Alg. 1, NEXT-1) and with static E:T:D
ratios, on one GPU with co-located instances (E x1, T x3, D x1).  Reports the throughput of
each phase, the controller's decisions (time, action, ratio, measured u/q/d per stage) and
that every request completed.

    python tools/workload_shift.py --out gpurun_out/workload_shift.json
"""
import argparse
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_25550_b200 import binding as B  # noqa: E402
from synth.configs import CONFIGS  # noqa: E402

INST = [(0, B.DF_E), (0, B.DF_T), (0, B.DF_T), (0, B.DF_T), (0, B.DF_D)]


def run(cfg, phases, mode, delta_s):
    """mode: 'controller' or a static (gE, gT, gD)."""
    g = B.make_graph(cfg, INST, max_steps=max(s for s, _ in phases), G=5)
    out = {"mode": mode if isinstance(mode, str) else "static %d:%d:%d" % mode, "phases": []}
    with B.Context(g) as c:
        c.submit(phases[0][0], cfg.shift, 99999)  # warm-up (not timed)
        while not c.poll(1, 120000):
            pass
        torch.cuda.synchronize()
        if mode == "controller":
            c.sched_start(B.sched_cfg(delta_s=delta_s, G=5))
        else:
            c.set_ratio(*mode)
        t_start = time.perf_counter()
        seed = 0
        done = []
        for steps, n in phases:
            t0 = time.perf_counter()
            tags = list(range(seed, seed + n))
            seed += n
            for s in tags:
                while c.submit(steps, cfg.shift, s, user_tag=s)[0] != B.DF_OK:
                    done += c.poll(32, 5)
            got = [x for x in done if x.user_tag in set(tags)]
            while len(got) < n:
                more = c.poll(32, 120000)
                done += more
                got += [x for x in more if x.user_tag in set(tags)]
            wall = time.perf_counter() - t0
            out["phases"].append({"steps": steps, "requests": n, "req_per_s": n / wall, "wall_s": wall})
        if mode == "controller":
            time.sleep(delta_s * 1.5)
            c.sched_stop()
            out["decisions"] = [{"t": round(ev.t - 0.0, 3), "action": int(ev.action), "stage": int(ev.stage),
                                 "g": list(ev.g), "u": [round(v, 3) for v in ev.m.u], "q": list(ev.m.q),
                                 "d_s": [round(v, 4) for v in ev.m.d]} for ev in c.sched_log()]
        out["all_completed"] = sorted(x.user_tag for x in done) == list(range(seed))
        out["total_s"] = time.perf_counter() - t_start
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="image")
    ap.add_argument("--heavy-steps", type=int, default=28)
    ap.add_argument("--light-steps", type=int, default=1)
    ap.add_argument("--heavy", type=int, default=18)
    ap.add_argument("--light", type=int, default=90)
    ap.add_argument("--delta", type=float, default=1.0, help="controller period (s); the paper uses 2 s")
    ap.add_argument("--out", default="gpurun_out/workload_shift.json")
    a = ap.parse_args()
    cfg = CONFIGS[a.config]
    phases = [(a.heavy_steps, a.heavy), (a.light_steps, a.light)]
    res = {"config": cfg.name, "layout": "E x1, T x3, D x1 co-located on GPU 0", "phases": phases, "runs": []}
    for mode in ("controller", (1, 3, 1), (1, 1, 1)):
        r = run(cfg, phases, mode, a.delta)
        res["runs"].append(r)
        print(json.dumps({k: v for k, v in r.items() if k != "decisions"}), flush=True)
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
