"""CPU multi-process tests of the N > 1 host logic (gloo, world_size 2): the
shared-memory FAA metadata ring between two processes, the stage layouts, and the
max-over-ranks timing reduction bench.py uses."""
import os
import socket
import uuid

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _ring_worker(rank, world, port, name, n, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import ctypes
    from paper_2605_25550_b200 import binding
    lib = binding.load()
    cs, ok = ctypes.c_uint64(), ctypes.c_int32()
    dist.barrier()
    st = lib.df_ring_selftest(name.encode(), rank, n, ctypes.byref(cs), ctypes.byref(ok))
    t = torch.tensor([st, cs.value, ok.value], dtype=torch.int64)
    out = [torch.zeros(3, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(out, t)
    # max-over-ranks reduction as bench.py does it
    ms = torch.tensor([10.0 * (rank + 1)], dtype=torch.float64)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    if rank == 0:
        q.put(([o.tolist() for o in out], float(ms)))
    dist.destroy_process_group()


@pytest.fixture(scope="module")
def lib_built():
    from paper_2605_25550_b200 import binding
    if not os.path.exists(binding.LIB_PATH):
        from paper_2605_25550_b200 import build
        build.build()
    return True


@pytest.mark.parametrize("n", [1, 64, 5000])
def test_shm_faa_ring_two_processes(lib_built, n):
    ctxm = mp.get_context("spawn")
    q = ctxm.Queue()
    name = f"/df_test_{uuid.uuid4().hex[:12]}"
    port = _free_port()
    procs = [ctxm.Process(target=_ring_worker, args=(r, 2, port, name, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    res, ms = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (st0, sum0, _), (st1, sum1, fifo1) = res
    assert st0 == 0 and st1 == 0
    assert sum0 == sum1 == n * (n - 1) // 2      # conservation: the same multiset
    assert fifo1 == 1                            # single-producer FIFO order preserved
    assert ms == 20.0                            # max over ranks


def test_layouts():
    from paper_2605_25550_b200 import layouts as L
    from paper_2605_25550_b200.binding import DF_E, DF_T, DF_D
    for n in (1, 2, 4, 8):
        inst = L.partitioned(n)
        gE, gT, gD = L.ratio(inst)
        assert gE == 1 and gD == 1 and gT == n
        assert {i[2] for i in inst} == set(range(n))         # every rank hosts an instance
        assert L.ranks_of(inst, DF_E) == [0] and L.ranks_of(inst, DF_D) == [n - 1]
    inst = L.partitioned(8, exclusive=True)
    assert L.ratio(inst) == (1, 6, 1)                        # the paper's 1:6:1
    assert sum(L.ratio(inst)) <= 8                            # Eq. 1
    with pytest.raises(ValueError):
        L.partitioned(2, exclusive=True)


def test_layouts_colocated_dit_instances():
    """Several DiT instances per GPU (bench --t-per-gpu): every GPU gets t instances of T,
    E stays on GPU 0 and D on the last GPU; ratios follow."""
    from paper_2605_25550_b200 import layouts as L
    from paper_2605_25550_b200.binding import DF_E, DF_T, DF_D
    inst = L.partitioned(1, t_per_gpu=2)
    assert L.ratio(inst) == (1, 2, 1) and all(i[2] == 0 for i in inst)
    inst = L.partitioned(4, t_per_gpu=3)
    assert L.ratio(inst) == (1, 12, 1)
    assert sorted({i[2] for i in inst if i[1] == DF_T}) == [0, 1, 2, 3]
    assert all(sum(1 for i in inst if i[1] == DF_T and i[2] == r) == 3 for r in range(4))
    assert L.ranks_of(inst, DF_E) == [0] and L.ranks_of(inst, DF_D) == [3]
    inst = L.partitioned(8, exclusive=True, t_per_gpu=2)
    assert L.ratio(inst) == (1, 12, 1) and L.ranks_of(inst, DF_T) == list(range(1, 7))
    with pytest.raises(ValueError):
        L.partitioned(2, t_per_gpu=0)
