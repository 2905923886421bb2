"""One process per instance group over the shared-memory plane + CUDA IPC (the N > 1
path), exercised on ONE GPU with two processes: rank 0 hosts E and T0, rank 1 hosts T1
and D, so requests cross the process boundary on both edges (E -> T1, T0 -> D)."""
import ctypes
import os
import socket
import uuid

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, shm, seeds, mode, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2605_25550_b200 import binding as B, layouts
    from synth.configs import TINY
    inst = layouts.partitioned(world)
    g = B.make_graph(TINY, inst, rank=rank, world=world, shm_name=shm, handoff_mode=mode,
                     chunk_bytes=(64, 256))
    c = B.Context(g)
    dist.barrier()
    got = {}
    if rank == 0:
        dummy = np.zeros(TINY.out_shape, np.float32)
        for s in seeds:
            st, _ = c.submit(TINY.steps, TINY.shift, s, out_host=dummy, user_tag=s)
            assert st == B.DF_OK
    if rank == world - 1:
        comps = []
        while len(comps) < len(seeds):
            for x in c.poll(8, timeout_ms=60000):
                assert x.out_view and x.out_view_bytes == np.prod(TINY.out_shape) * 4
                buf = (ctypes.c_char * x.out_view_bytes).from_address(x.out_view)
                got[int(x.user_tag)] = (np.frombuffer(bytes(buf), np.float32).reshape(TINY.out_shape).copy(),
                                        list(x.inst), float(x.exposed_ms[1]),
                                        (x.hash_src[1], x.hash_dst[1]))
                comps.append(x)
        q.put(got)
    dist.barrier()
    c.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", [4, 4 | 1])  # DF_HASH, DF_HASH|DF_SYNC
def test_two_process_pipeline_matches_oracle_and_single_process(mode):
    import torch.multiprocessing as mp
    from oracle import params as OP, stages
    from synth.configs import TINY
    from gpu_util import rel_l2, make_ctx
    seeds = [11, 12, 13, 14, 15]
    ctxm = mp.get_context("spawn")
    q = ctxm.Queue()
    shm = f"/df_gpu_{uuid.uuid4().hex[:10]}"
    procs = [ctxm.Process(target=_worker, args=(r, 2, _port(), shm, seeds, mode, q)) for r in range(2)]
    # both ranks need the same port: rebuild with a shared one
    port = _port()
    procs = [ctxm.Process(target=_worker, args=(r, 2, port, shm, seeds, mode, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert sorted(got) == seeds                               # conservation, no duplicates
    assert {tuple(v[1][1:2]) for v in got.values()} == {(1,), (2,)}  # both T instances served
    P = OP.Params(TINY, 0)
    single = {}
    with make_ctx(TINY, handoff_mode=mode, chunk_bytes=(64, 256)) as c:
        outs = {s: np.zeros(TINY.out_shape, np.float32) for s in seeds}
        for s in seeds:
            c.submit(TINY.steps, TINY.shift, s, out_host=outs[s], user_tag=s)
        n = 0
        while n < len(seeds):
            n += len(c.poll(8, 60000))
        single = outs
    for s in seeds:
        out, inst, exposed, (hs, hd) = got[s]
        assert hs == hd != 0                                  # T->D tensor hash check
        want = stages.request(P, TINY, seed=s)["out"]
        assert rel_l2(out, want) <= 3e-2
        assert np.array_equal(out, single[s])                 # bit-identical to the 1-process run


def _jitter_worker(rank, world, port, shm, seeds, mode, d, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["DF_JITTER_EDGES"] = "2"  # delay the T->D transfers only
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2605_25550_b200 import binding as B, layouts
    from synth.configs import TINY
    g = B.make_graph(TINY, layouts.partitioned(world), rank=rank, world=world, shm_name=shm, handoff_mode=mode,
                     chunk_bytes=(64, 256), jitter=(1.0, d, 3))
    c = B.Context(g)
    dist.barrier()
    if rank == 0:
        for s in seeds:
            assert c.submit(TINY.steps, TINY.shift, s, user_tag=s)[0] == B.DF_OK
    if rank == world - 1:
        got = []
        while len(got) < len(seeds):
            for x in c.poll(8, timeout_ms=60000):
                got.append((int(x.user_tag), int(x.inst[1]), float(x.t_end[1]), float(x.exposed_ms[1]),
                            float(x.xfer_ms[1]), float(x.xfer_ms[0]), x.hash_src[0] == x.hash_dst[0] != 0,
                            x.hash_src[1] == x.hash_dst[1] != 0))
        q.put(got)
    dist.barrier()
    c.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", [4, 4 | 1])  # DF_HASH (async), DF_HASH|DF_SYNC
def test_two_process_handoff_is_asynchronous(mode):
    """P:L154 / P:L513 on the one-process-per-GPU path: every T->D transfer is held back by
    d = 0.2 s on the producer's comm stream.  Asynchronous: a T instance computes its next
    request without waiting for the delayed send (its two requests finish far less than d
    apart; the delay shows up only as the decoder's exposed wait).  DF_SYNC: the T
    compute stream waits for each delivery, so its second request finishes >= d after the
    first.  Hashes match on both edges; transfers are timed on the consumer's clock."""
    import torch.multiprocessing as mp
    d = 0.2
    seeds = [21, 22, 23, 24]
    ctxm = mp.get_context("spawn")
    q = ctxm.Queue()
    shm = f"/df_gpu_{uuid.uuid4().hex[:10]}"
    port = _port()
    procs = [ctxm.Process(target=_jitter_worker, args=(r, 2, port, shm, seeds, mode, d, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert sorted(g[0] for g in got) == seeds
    by_t = {}
    for tag, t_inst, t_end_t, exposed1, xfer1, xfer0, h0, h1 in got:
        assert h0 and h1
        assert 0 < xfer0 < 0.5 * d * 1e3 and 0 < xfer1 < 0.5 * d * 1e3  # copies timed without the delay
        by_t.setdefault(t_inst, []).append(t_end_t)
    # D stalled on delayed data (its decodes are serial, so a stall that overlaps an earlier
    # request's is counted once, on that request)
    assert max(g[3] for g in got) >= 0.8 * d * 1e3
    assert len(by_t) == 2
    for t_inst, ends in by_t.items():
        ends.sort()
        gap = ends[1] - ends[0]
        if mode & 1:
            assert gap >= 0.8 * d, (t_inst, gap)
        else:
            assert gap < 0.25 * d, (t_inst, gap)


def _sched_worker(rank, world, port, shm, q):
    import sys
    import time
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2605_25550_b200 import binding as B
    from synth.configs import TINY
    # rank 0: E0, T1; rank 1: T2, D3, and a second encoder E4 (inactive until scaled out)
    inst = [(0, B.DF_E, 0), (0, B.DF_T, 0), (0, B.DF_T, 1), (0, B.DF_D, 1), (0, B.DF_E, 1)]
    g = B.make_graph(TINY, inst, rank=rank, world=world, shm_name=shm, chunk_bytes=(64, 256))
    c = B.Context(g)
    dist.barrier()
    res = {}

    def drain(n):
        got = []
        while len(got) < n:
            got += [(int(x.user_tag), int(x.inst[0]), x.hash_src[0] == x.hash_dst[0] != 0)
                    for x in c.poll(16, timeout_ms=60000)]
        return got

    if rank == 0:
        assert c.set_ratio(1, 2, 1) == B.DF_OK                     # E4 (rank 1) stops pulling
    dist.barrier()
    # phase A: one encoder, no controller.  Phase B: the Alg. 1 controller on rank 0 with a
    # hair-trigger scale-out rule (u > 0, q > 0, d rising) sees the encoder queue of a request
    # burst and scales E out -- to the encoder hosted by rank 1.  Phase C: back to one encoder
    # by an explicit df_set_ratio.
    for phase, seeds in (("A", list(range(100, 140))), ("B", list(range(200, 400))), ("C", list(range(500, 540)))):
        if rank == 0:
            if phase == "B":
                c.sched_start(B.sched_cfg(delta_s=0.02, U_high=0.0, U_low=-1.0, Q_high=0, move_budget=0))
            if phase == "C":
                c.sched_stop()
                assert c.set_ratio(1, 2, 1) == B.DF_OK
            for k, s in enumerate(seeds):
                while c.submit(TINY.steps, TINY.shift, s, user_tag=s)[0] != B.DF_OK:
                    time.sleep(0.001)
                if phase == "B" and k % 25 == 24:
                    time.sleep(0.01)  # spread the burst over several controller ticks
        if rank == 1:
            res[phase] = drain(len(seeds))
        dist.barrier()
    if rank == 0:
        log = c.sched_log()
        res["log"] = [(e.action, e.stage, tuple(e.g), tuple(e.m.u), tuple(e.m.q)) for e in log]
    objs = [None, None]
    dist.all_gather_object(objs, res)
    if rank == 0:
        q.put({**objs[0], **objs[1]})
    dist.barrier()
    c.close()
    dist.destroy_process_group()


def test_two_process_controller_and_encoder_scale_out():
    """NEXT-1 across processes (P:L326-357 on the one-process-per-GPU path): the request ring,
    the allocation g_s and every instance's busy time live in the shared plane.  The Alg. 1
    controller on rank 0 measures all instances (rank 1's D included) and, when the encoder
    queue builds up, scales E out to the encoder hosted by rank 1, which then pulls
    requests submitted on rank 0; an explicit df_set_ratio scales it back in.  No request is
    lost and every handoff hash matches."""
    import torch.multiprocessing as mp
    ctxm = mp.get_context("spawn")
    q = ctxm.Queue()
    shm = f"/df_gpu_{uuid.uuid4().hex[:10]}"
    port = _port()
    procs = [ctxm.Process(target=_sched_worker, args=(r, 2, port, shm, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    a, b, cc = res["A"], res["B"], res["C"]
    assert sorted(x[0] for x in a) == list(range(100, 140)) and sorted(x[0] for x in b) == list(range(200, 400))
    assert sorted(x[0] for x in cc) == list(range(500, 540))
    assert all(x[2] for x in a + b + cc)
    assert {x[1] for x in a} == {0} and {x[1] for x in cc} == {0}   # one encoder
    assert 4 in {x[1] for x in b}                                  # the controller scaled out to rank 1's encoder
    log = res["log"]
    assert any(act == 1 and st == 0 for act, st, _, _, _ in log)   # logged as an E scale-out
    for action, st, g, u, qq in log:
        assert min(g) >= 1 and g[0] <= 2 and g[1] <= 2 and g[2] == 1
        assert all(0.0 <= x <= 1.0 for x in u)
    assert any(u[2] > 0 for _, _, _, u, _ in log)                 # the D on rank 1 is seen as busy


def _repurpose_worker(rank, world, port, shm, q):
    import sys
    import time
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2605_25550_b200 import binding as B, layouts
    from synth.configs import TINY
    inst = layouts.partitioned(world)  # rank 0: E0, T1; rank 1: T2, D3
    g = B.make_graph(TINY, inst, rank=rank, world=world, shm_name=shm, chunk_bytes=(64, 256))
    c = B.Context(g)
    dist.barrier()
    res = {}
    phases = (("A", None, list(range(10, 30))), ("B", (2, 1, 1), list(range(30, 50))),
              ("C", (1, 2, 1), list(range(50, 70))))
    for name, ratio, seeds in phases:
        if rank == 0:
            if ratio is not None:
                assert c.set_ratio(*ratio) == B.DF_OK
            for s in seeds:
                while c.submit(TINY.steps, TINY.shift, s, user_tag=s)[0] != B.DF_OK:
                    time.sleep(0.001)
        if rank == 1:
            got = []
            while len(got) < len(seeds):
                got += [(int(x.user_tag), tuple(int(v) for v in x.inst),
                         all(x.hash_src[e] == x.hash_dst[e] != 0 for e in range(2)))
                        for x in c.poll(16, timeout_ms=60000)]
            res[name] = got
        dist.barrier()
    if rank == 0:
        res["log"] = [(e.action, e.inst, e.from_stage, e.stage, e.cold_start_ms) for e in c.sched_log()]
    objs = [None, None]
    dist.all_gather_object(objs, res)
    if rank == 0:
        q.put({**objs[0], **objs[1]})
    dist.barrier()
    c.close()
    dist.destroy_process_group()


def test_two_process_repurposing():
    """Re-purposing on the one-process-per-GPU path ("Apply", P:L357 cold start): rank 0's
    df_set_ratio(2, 1, 1) drains its own DiT instance T1 and re-creates it as a second encoder
    (the shared routing stops sending it work, producers on every rank finish what they picked);
    df_set_ratio(1, 2, 1) turns it back into a DiT instance, which re-publishes its receive slots
    (rank 0's encoder re-opens them; rank 1's decoder keeps receiving from it).  No request is
    lost, hashes match, and every phase serves from the instances its allocation names."""
    import torch.multiprocessing as mp
    ctxm = mp.get_context("spawn")
    q = ctxm.Queue()
    shm = f"/df_gpu_{uuid.uuid4().hex[:10]}"
    port = _port()
    procs = [ctxm.Process(target=_repurpose_worker, args=(r, 2, port, shm, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for name, lo in (("A", 10), ("B", 30), ("C", 50)):
        got = res[name]
        assert sorted(x[0] for x in got) == list(range(lo, lo + 20)) and all(x[2] for x in got)
    assert {x[1][1] for x in res["A"]} == {1, 2}                   # two DiT instances
    assert {x[1][1] for x in res["B"]} == {2}                      # T1 is an encoder now
    assert {x[1][0] for x in res["B"]} <= {0, 1}
    assert {x[1][1] for x in res["C"]} == {1, 2}                   # and a DiT instance again
    log = [e for e in res["log"] if e[0] == 4]
    assert [(e[1], e[2], e[3]) for e in log] == [(1, 1, 0), (1, 0, 1)]
    assert all(e[4] > 0 for e in log)
