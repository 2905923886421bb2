"""Probe: does a sleeping host function (the jitter injector, `df::delay_ns`) on one stream
stall work on another stream of the same device?  Times a fixed GEMM loop on stream B with
and without a 150 ms host function queued on stream A, with B's loop optionally containing a
pageable host->device copy (what Model::prepare does for the sigma schedule).

    python tools/hostfn_probe.py
"""
import ctypes
import json
import os
import time

import numpy as np
import torch

LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2605_25550_b200", "libdf.so")


def main():
    lib = ctypes.CDLL(LIB)
    delay = getattr(lib, "_ZN2df8delay_nsEmP11CUstream_st")
    delay.argtypes = [ctypes.c_uint64, ctypes.c_void_p]
    delay.restype = ctypes.c_int
    a = torch.randn(4096, 4096, device="cuda", dtype=torch.bfloat16)
    sA, sB = torch.cuda.Stream(), torch.cuda.Stream()
    host = np.arange(64, dtype=np.float32)
    dev = torch.empty(64, device="cuda")
    res = {}

    def loop(n, pageable):
        with torch.cuda.stream(sB):
            for i in range(n):
                torch.mm(a, a)
                if pageable and i == n // 4:
                    dev.copy_(torch.from_numpy(host), non_blocking=True)  # pageable H2D

    for case in ("base", "hostfn", "base_pageable", "hostfn_pageable"):
        loop(20, False)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if case.startswith("hostfn"):
            assert delay(150_000_000, sA.cuda_stream) == 0
        t0 = time.perf_counter()
        e0.record(sB)
        loop(400, case.endswith("pageable"))
        e1.record(sB)
        t_enq = time.perf_counter() - t0
        torch.cuda.synchronize()
        res[case] = {"device_ms": e0.elapsed_time(e1), "host_enqueue_ms": t_enq * 1e3}
        print(case, res[case], flush=True)
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/hostfn_probe.json", "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
