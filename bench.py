#!/usr/bin/env python
"""Benchmark: requests/sec/box of the disaggregated E -> T -> D pipeline (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config image|video|mid|tiny]

One "step" = one request through every §8(a) row (E stand-in, E->T chunked handoff,
DiT prologue + S Euler steps, T->D chunked handoff, D stand-in) on the BASELINE
configs[1] workload: text-to-image 1024x1024 -> 4096 latent tokens, DiT hidden 3072 x 28
layers, 28 steps, bf16, random-init weights, synthetic requests.

N=1: E, T and D co-resident on GPU 0 (layout 1:1:1), requests pipelined through the async
handoff.  N>1 (torchrun, one process per GPU): stage-partitioned, E on GPU 0, D on GPU N-1
and a DiT instance on every GPU (1:N:1; --exclusive gives E and D GPUs of their own, the
paper's 1:6:1 at N=8); requests cross GPUs through the asynchronous chunked handoff
(shared-memory FAA metadata rings + CUDA IPC receive slots, copies over NVLink).  K
requests per DiT instance -> "scaling": "weak".  The process group (NCCL; gloo with
DF_BENCH_BACKEND=gloo) is plumbing only: barriers and the max-over-ranks reduction.

Prints ONE JSON line (rank 0).  --impl reference times the fp64 CPU oracle (the
reference arm for this tier) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from synth.configs import CONFIGS, with_layers  # noqa: E402

METRIC = "requests/sec/box at 1/2/4/8 B200; DiT step tensor-pipe %; exposed handoff ms"
UNIT = "requests/s"


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return {"hbm": j["hbm_gbs"], "bf16": j["bf16_tflops"], "bf16_sus": j.get("bf16_tflops_sustained", j["bf16_tflops"]),
                "src": "measured"}
    return {"hbm": 6650.0, "bf16": 1590.0, "bf16_sus": 1400.0, "src": "fallback"}


# ------------------------------------------------------------------ clocks sampler
class Clocks:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = max(mx, float(parts[2]))
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        load = [s for s in sm if s > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(load), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ oracle timing (reference arm / cpu_baseline)
def oracle_sample(cfg, reps=1):
    """Time the fp64 oracle on ONE DiT block with the workload's width (d, heads, f,
    L_txt) on a bounded token count (a 32x32 latent, N = 1024: ~10-30 s of CPU work);
    weights are generated beforehand (untimed).  Extrapolate by algorithmic FLOP:
    requests/s = (oracle FLOP/s on the sample) / (FLOP per request of the workload)."""
    import dataclasses
    import numpy as np
    from oracle import params as OP, dit
    from synth import inputs
    c1 = dataclasses.replace(with_layers(cfg, 1), F=1, H=min(cfg.H, 64), W=min(cfg.W, 64))
    P = OP.Params(c1, 0)
    for n in ("L0.mod", "L0.qkv_w", "L0.qkv_b", "L0.g_q", "L0.g_k", "L0.o_w", "L0.o_b", "L0.g_n3", "L0.cq_w",
              "L0.cq_b", "L0.g_cq", "L0.co_w", "L0.co_b", "L0.w1", "L0.b1", "L0.w3", "L0.b3", "L0.w2", "L0.b2"):
        P[n]
    r = inputs.residual(c1, 1).astype(np.float64)
    rr = np.random.default_rng(0)
    kv = (rr.standard_normal((cfg.L_txt, cfg.d)), rr.standard_normal((cfg.L_txt, cfg.d)))
    e6 = rr.standard_normal((6, cfg.d)) * 0.1
    pos = dit.token_positions(c1)
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        dit.block(P, c1, 0, r, e6, kv, pos)
        times.append(time.perf_counter() - t0)
    t = min(times)
    block_flops = (c1.flops_per_step() - 4 * c1.N * c1.P * c1.d) / c1.layers
    rate = block_flops / t
    try:
        from threadpoolctl import threadpool_info
        cores = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        cores = os.cpu_count()
    return {"t_block_s": t, "value": rate / cfg.flops_per_request(), "cores": cores, "gflops": rate / 1e9,
            "sample": f"1 DiT block at the {cfg.name} width (d={cfg.d}, heads={cfg.heads}, f={cfg.ffn}, "
                      f"L_txt={cfg.L_txt}) on N={c1.N} tokens, fp64 numpy oracle ({rate / 1e9:.1f} GFLOP/s), "
                      f"extrapolated by FLOP to one {cfg.name} request ({cfg.flops_per_request():.3e} FLOP)"}


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    for _ in range(args.warmup):
        pass  # the oracle has no warm state worth warming; keep the contract's shape
    vals, blocks = [], []
    t_all = time.perf_counter()
    for _ in range(args.steps):
        s = oracle_sample(cfg)
        vals.append(s["value"])
        blocks.append(s["t_block_s"])
    wall = time.perf_counter() - t_all
    v = statistics.median(vals)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 / v, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_name(cfg)},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": s["cores"], "kind": "oracle", "sample": s["sample"]},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "oracle_block_s": statistics.median(blocks), "wall_s": wall}
    print(json.dumps(line), flush=True)


def workload_name(cfg):
    if cfg.name == "image":
        return "text-to-image 1024x1024 -> 4096 latent tokens, DiT hidden 3072 x28 layers, 28 Euler steps (BASELINE configs[1])"
    if cfg.name == "video":
        return "text-to-video 81x480x832 -> 32760 latent tokens, DiT hidden 5120 x40 layers, 50 Euler steps (BASELINE configs[2])"
    if cfg.name == "video_i2v":
        return (f"image-to-video 81x480x832 -> 32760 latent tokens (+ y 20 channels, 257 CLIP tokens), DiT hidden "
                f"5120 x40 layers, {cfg.steps} Euler steps (the paper's Wan2.2 I2V workload, P:L441; not a BASELINE config)")
    return f"{cfg.name}: N={cfg.N} d={cfg.d} layers={cfg.layers} steps={cfg.steps}"


# ------------------------------------------------------------------ our arm
def summarize(comps, ecomps=()):
    """Per-request pipeline numbers from df_completion records (D rank)."""
    lat = [(c.t_done - c.t_submit) * 1000.0 for c in comps]
    exposed = [c.exposed_ms[0] + c.exposed_ms[1] for c in comps]
    med = statistics.median

    def pos(v):
        v = [x for x in v if x > 0]
        return med(v) if v else -1.0
    return {
        "t_ms": med(c.stage_ms[1] for c in comps),
        "lat": med(lat), "exp_med": med(exposed), "exp_max": max(exposed),
        "exp_frac": med(exposed) / med(lat),
        "exp_edge": [med(c.exposed_ms[0] for c in comps), med(c.exposed_ms[1] for c in comps)],
        "xfer": [pos([c.xfer_ms[0] for c in comps]), pos([c.xfer_ms[1] for c in comps])],
        "overlap": [med(c.overlap_ms[0] for c in comps), med(c.overlap_ms[1] for c in comps)],
        "hash_ok": all(c.hash_src[e] == c.hash_dst[e] != 0 for c in list(comps) + list(ecomps) for e in range(2)),
        "n": len(comps), "t_inst": sorted({int(c.inst[1]) for c in comps}),
        # per-instance stage times for Eq. 6: E host enqueue time (E never waits on the
        # device), T and D device time of one request
        "T_s": [med((c.t_end[0] - c.t_start[0]) for c in comps), med(c.stage_ms[1] for c in comps) * 1e-3,
                med(c.stage_ms[2] for c in comps) * 1e-3]}


def eq6_record(g, T, value):
    """P14 (Eq. 6): the pipeline's throughput bound min_s g_s / T_s from the
    measured per-instance stage times, and the measured whole-job rate as a fraction of it."""
    rates = [g[s] / T[s] if T[s] > 0 else float("inf") for s in range(3)]
    b = min(range(3), key=lambda s: rates[s])
    return {"g": list(g), "T_s": T, "bound_req_s": rates[b], "bottleneck": "ETD"[b], "measured_over_bound": value / rates[b]}


def roofline(kstats, peaks, traffic, config):
    """Roofline of the kernel class with the largest measured time share (this rank's DiT
    instance, per-launch CUDA events on its stream)."""
    dom = max(kstats, key=lambda k: kstats[k]["ms"])
    ks = kstats[dom]
    avg_ms = ks["ms"] / max(ks["launches"], 1)
    if ks["flops"] > 0:
        ach = (ks["flops"] / ks["launches"]) / (avg_ms / 1000.0) / 1e12
        # the sustained figure (cuBLAS 8192^3 back to back, deepest power-cap clocks) is the
        # denominator for a kernel timed inside a long step unless the kernel beats it; then the
        # burst figure is the ceiling that still holds
        if ach <= peaks["bf16_sus"]:
            pk, note = peaks["bf16_sus"], f"{peaks['src']} sustained cuBLAS bf16 (kernel timed inside a long step)"
        else:
            pk = peaks["bf16"]
            note = (f"{peaks['src']} burst cuBLAS bf16: the kernel exceeds the sustained figure "
                    f"({peaks['bf16_sus']:.1f}), which was measured at lower power-capped clocks")
        roof = {"bound": "tensor", "achieved": ach, "peak": pk, "unit": "TFLOP/s",
                "frac": ach / pk, "traffic": traffic, "kernel": dom,
                "avg_launch_us": avg_ms * 1000.0, "launches": ks["launches"], "peak_note": note}
    else:
        ach = (ks["bytes"] / ks["launches"]) / (avg_ms / 1000.0) / 1e9
        roof = {"bound": "hbm", "achieved": ach, "peak": peaks["hbm"], "unit": "GB/s", "frac": ach / peaks["hbm"],
                "traffic": traffic, "kernel": dom, "avg_launch_us": avg_ms * 1000.0, "launches": ks["launches"],
                "peak_note": f"{peaks['src']} HBM copy"}
    if roof["traffic"] is None:  # committed ncu capture of this kernel at this config, if any
        try:
            tj = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
            ent = tj.get(config, {}).get(dom)
            if ent:
                roof["traffic"] = ent["bytes"]
                roof["traffic_source"] = ent["source"]
        except (OSError, ValueError):
            pass
    return roof


def kernel_tables(kstats):
    tot = sum(v["ms"] for v in kstats.values()) or 1.0
    shares = {k: round(v["ms"] / tot, 4) for k, v in kstats.items() if v["ms"] > 0}
    gfl = {k: round((v["flops"] / v["ms"] / 1e9), 1) for k, v in kstats.items() if v["ms"] > 0 and v["flops"] > 0}
    return shares, gfl


def payload_bytes(cfg):
    """Per-request payloads of the two edges (E->T: ctx [| clip | y]; T->D: the fp32 latent)."""
    e2t = cfg.L_txt * cfg.d_txt * 2 + (((cfg.L_img * cfg.d_img * 2 + 15) // 16) * 16 +
                                       cfg.C_y * cfg.F * cfg.H * cfg.W * 4 if cfg.C_y else 0)
    return e2t, cfg.latent_elems * 4


def handoff_record(cfg, summary):
    e2t, t2d = payload_bytes(cfg)
    return {"exposed_ms_median": summary["exp_med"], "exposed_ms_max": summary["exp_max"],
            "exposed_ms_median_per_edge": summary["exp_edge"],
            "exposed_frac_of_latency": summary["exp_frac"], "xfer_ms_median": summary["xfer"],
            "payload_bytes": [e2t, t2d],
            "xfer_gbps": [(e2t / summary["xfer"][0] / 1e6) if summary["xfer"][0] > 0 else None,
                          (t2d / summary["xfer"][1] / 1e6) if summary["xfer"][1] > 0 else None],
            "consumer_overlap_ms_median": summary["overlap"],
            "latency_ms_median": summary["lat"], "hash_match": summary["hash_ok"],
            "dit_instances_used": summary["t_inst"]}


def sub_record(args, peaks, local, cfg, precision, warm, n, what):
    """A further workload through the same E -> T -> D pipeline on this GPU (E:T:D 1:1:1):
    `warm` warm-up requests, then `n` timed requests with inputs device-resident (tokens and
    noise from the seed), the DiT step's roofline and the clocks sampled in the timed region."""
    import torch
    from paper_2605_25550_b200 import binding as B, layouts
    inst = layouts.partitioned(1)
    g = B.make_graph(cfg, inst, precision=precision, weight_seed=0, chunk_bytes=(args.chunk_ctx, args.chunk_lat),
                     n_slots=2, handoff_mode=B.DF_ASYNC | B.DF_HASH, ring_capacity=64, max_steps=cfg.steps)
    ctx = B.Context(g)
    stream = torch.cuda.current_stream()

    def batch(k, seed0):
        for j in range(k):
            while ctx.submit(cfg.steps, cfg.shift, seed0 + j, user_tag=seed0 + j)[0] != B.DF_OK:
                time.sleep(0.01)
        comps = []
        while len(comps) < k:
            comps += ctx.poll(16, timeout_ms=1000)
        return comps

    try:
        batch(warm, 5000)
        torch.cuda.synchronize()
        ctx.profile(4, True)
        l0 = ctx.launch_count()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with Clocks(local) as clk:
            torch.cuda.synchronize()
            ev0.record(stream)
            comps = batch(n, 6000)
            ev1.record(stream)
            ev1.synchronize()
        ms = ev0.elapsed_time(ev1)
        launches = ctx.launch_count() - l0
        kstats = ctx.kernel_stats()
        ctx.profile(False, False)
    finally:
        ctx.close()
    summ = summarize(comps)
    tflop = cfg.flops_per_request() / 1e12
    tfs = tflop / (summ["t_ms"] / 1000.0)
    shares, gfl = kernel_tables(kstats)
    return {"what": what, "workload": workload_name(cfg), "E:T:D": "1:1:1", "requests": n, "warmup_requests": warm,
            "value": n / (ms / 1000.0), "unit": UNIT, "ms_per_request": ms / n, "gpu_launches": launches,
            "dit_step": {"tflop_per_request": tflop, "tflop_per_step": cfg.flops_per_step() / 1e12,
                         "t_stage_ms_median": summ["t_ms"], "achieved_tflops": tfs,
                         "frac_of_sustained_peak": tfs / peaks["bf16_sus"], "frac_of_burst_peak": tfs / peaks["bf16"]},
            "roofline": roofline(kstats, peaks, None, cfg.name),
            "clocks": clk.summary(),
            "handoff": handoff_record(cfg, summ),
            "eq6": eq6_record((1, 1, 1), summ["T_s"], n / (ms / 1000.0)),
            "kernel_time_share": shares, "kernel_gflops": gfl}


def run_ours(args, cfg):
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2605_25550_b200 import binding as B, layouts

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    local = int(os.environ.get("DF_BENCH_DEVICE", local))  # tests: several ranks on one GPU
    backend = os.environ.get("DF_BENCH_BACKEND", "nccl")
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", init_method="env://", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend, init_method="env://")
    torch.cuda.set_device(local)
    red_dev = "cuda" if backend == "nccl" else "cpu"
    peaks = load_peaks()

    # Layout: N = 1 -> E+T+D on GPU 0; N > 1 -> one process per GPU, a DiT
    # instance on every GPU, E on GPU 0 and D on GPU N-1 (E:T:D = 1:N:1), requests cross
    # GPUs through the async chunked handoff (shared-memory rings + CUDA IPC over NVLink).
    inst = [(local if i[2] == rank else 0, i[1], i[2])
            for i in layouts.partitioned(world, args.exclusive, args.t_per_gpu)]
    shm = f"/df_bench_{os.environ.get('MASTER_PORT', '0')}_{os.getuid()}"
    prec = {"fp8": B.DF_FP8, "mxfp8": B.DF_MXFP8}.get(args.precision, B.DF_BF16)
    g = B.make_graph(cfg, inst, precision=prec, weight_seed=0,
                     chunk_bytes=(args.chunk_ctx, args.chunk_lat), n_slots=2,
                     handoff_mode=B.DF_ASYNC | B.DF_HASH, ring_capacity=256, max_steps=cfg.steps,
                     rank=rank, world=world, shm_name=shm if world > 1 else "")
    ctx = B.Context(g)
    stream = torch.cuda.current_stream()
    e_rank, d_rank = layouts.ranks_of(inst, B.DF_E)[0], layouts.ranks_of(inst, B.DF_D)[0]
    n_t = layouts.ratio(inst)[1]

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    def run_batch(n, seed0, with_host_io=False):
        """Submit n requests on the E rank; collect n completions on the D rank."""
        comps, outs = [], []
        if rank == e_rank:
            rng = np.random.default_rng(seed0)
            dummy = np.empty(cfg.out_shape, np.float32) if with_host_io else None
            for k in range(n):
                ids = rng.integers(0, cfg.vocab, cfg.L_txt, dtype=np.int32) if with_host_io else None
                while True:
                    st, _ = ctx.submit(cfg.steps, cfg.shift, seed0 + k, out_host=dummy, token_ids=ids,
                                       user_tag=seed0 + k)
                    if st == B.DF_OK:
                        break
                    if rank == d_rank:
                        comps += ctx.poll(16, timeout_ms=5)
                    else:
                        time.sleep(0.002)
        if rank == d_rank:
            while len(comps) < n:
                got = ctx.poll(16, timeout_ms=1000)
                if with_host_io:  # the decoded images are host-resident on this rank
                    for x in got:
                        outs.append(np.ctypeslib.as_array(
                            (np.ctypeslib.ctypes.c_float * (x.out_view_bytes // 4)).from_address(x.out_view)).sum())
                comps += got
        return comps

    n_total = args.steps * n_t          # weak scaling: K requests per DiT instance
    run_batch(args.warmup * n_t, 1000)
    barrier()
    # ---- timed region (inputs device-resident: tokens and noise from seeds on the device)
    # per-kernel CUDA events on every 4th denoising step of the timed region (every step's
    # ~300 event pairs would otherwise add their own GPU commands to the measured time)
    ctx.profile(4, True)
    l0 = ctx.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        barrier()
        ev0.record(stream)
        comps = run_batch(n_total, 2000)
        if world > 1:
            dist.barrier()  # the D rank's completion of the last request ends the region
        ev1.record(stream)
        ev1.synchronize()
    ms = ev0.elapsed_time(ev1)
    launches = ctx.launch_count() - l0
    kstats = ctx.kernel_stats()
    ctx.profile(False, False)
    # ---- e2e: host token ids in, host images out, through the public API
    out_bytes = int(np.prod(cfg.out_shape)) * 4
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    ecomps = run_batch(n_total, 3000, with_host_io=True)
    if world > 1:
        dist.barrier()
    e1.record(stream)
    e1.synchronize()
    ems = e0.elapsed_time(e1)

    # ---- max over ranks; completions live on the D rank
    t = torch.tensor([ms, ems], device=red_dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms, ems = float(t[0]), float(t[1])
    launches_t = torch.tensor([launches], device=red_dev, dtype=torch.int64)
    if world > 1:
        dist.all_reduce(launches_t)
    summary = summarize(comps, ecomps) if rank == d_rank else None
    if world > 1:
        objs = [None] * world
        dist.all_gather_object(objs, summary)
        summary = objs[d_rank]
    value = n_total / (ms / 1000.0)
    e2e = n_total / (ems / 1000.0)
    dit_tflop = cfg.flops_per_request() / 1e12
    dit_tflops = dit_tflop / (summary["t_ms"] / 1000.0)
    roof = roofline(kstats, peaks, args.traffic, args.config)
    shares, tput_kind = kernel_tables(kstats)
    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        ctx.close()
        return
    ctx.close()
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        s = oracle_sample(cfg)
        cpu = {"value": s["value"], "unit": UNIT, "cores": s["cores"], "kind": "oracle", "sample": s["sample"]}
    video = fp8 = mxfp8 = None
    if world == 1 and args.config == "image" and args.video_requests > 0 and prec == B.DF_BF16:
        # the north_star's headline shape (BASELINE configs[2], C3): 1 warm-up + K timed 50-step requests
        video = sub_record(args, peaks, local, CONFIGS["video"], B.DF_BF16, 1, args.video_requests,
                           "text-to-video (C3) through the same pipeline, bf16")
    if world == 1 and args.config == "image" and args.fp8_requests > 0 and prec == B.DF_BF16:
        # NEXT-4 (R29): the same image workload with the FP8 step mode (QKV, cross-Q and MLP-up
        # on e4m3 operands); dtype stays bf16 for the headline above -- this is a separate line
        fp8 = sub_record(args, peaks, local, cfg, B.DF_FP8, args.warmup, args.fp8_requests,
                         "text-to-image (C2), FP8 step mode (R29): e4m3 operands on the six block GEMMs")
        fp8["dtype"] = "e4m3 x e4m3 -> fp32 (six block GEMMs, per-row / per-tensor scales), bf16 elsewhere"
    if world == 1 and args.config == "image" and args.mxfp8_requests > 0 and prec == B.DF_BF16:
        # NEXT-4 (R31): the same image workload with MXFP8 block-scaled operands on the six block GEMMs
        mxfp8 = sub_record(args, peaks, local, cfg, B.DF_MXFP8, args.warmup, args.mxfp8_requests,
                           "text-to-image (C2), MXFP8 step mode (R31): OCP MX e4m3 block-32 scales, six block GEMMs")
        mxfp8["dtype"] = "MXFP8 (e4m3 + E8M0 block-32 scales) -> fp32 (six block GEMMs), bf16 elsewhere"
    gE, gT, gD = layouts.ratio(inst)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / n_total, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": {B.DF_BF16: "bf16", B.DF_FP8: "e4m3 block GEMMs (R29), bf16 elsewhere"}.get(
            prec, "MXFP8 block GEMMs (R31), bf16 elsewhere"), "data": "synthetic",
        "config": {"workload": workload_name(cfg),
                   "layout": ("E+T+D co-resident on GPU 0" if world == 1 else
                              f"stage-partitioned, one process per GPU: E on GPU 0, D on GPU {world - 1}, "
                              f"a DiT instance on {'every' if not args.exclusive else 'each other'} GPU; "
                              "cross-GPU handoff via shared-memory FAA rings + CUDA IPC slots"),
                   "E:T:D": f"{gE}:{gT}:{gD}", "requests": n_total, "requests_per_dit_instance": args.steps,
                   "steps_per_request": cfg.steps, "chunk_bytes": [args.chunk_ctx, args.chunk_lat],
                   "l2": "inputs larger than L2: the DiT streams 8.5 GB of weights per denoising step"
                         if cfg.name == "image" else "weights per step exceed L2"},
        "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": cfg.L_txt * 4, "d2h_bytes_per_step": out_bytes},
        "gpu_launches": int(launches_t.item()),
        "roofline": roof,
        "cpu_baseline": cpu,
        "clocks": clk.summary(),
        "dit_step": {"tflop_per_request": dit_tflop, "t_stage_ms_median": summary["t_ms"],
                     "achieved_tflops": dit_tflops, "frac_of_sustained_peak": dit_tflops / peaks["bf16_sus"],
                     "frac_of_burst_peak": dit_tflops / peaks["bf16"]},
        "handoff": handoff_record(cfg, summary),
        "eq6": eq6_record((gE, gT, gD), summary["T_s"], value),
        "kernel_time_share": shares,
        "kernel_gflops": tput_kind,
    }
    if video is not None:
        line["video"] = video
    if fp8 is not None:
        line["fp8"] = fp8
    if mxfp8 is not None:
        line["mxfp8"] = mxfp8
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="image", choices=sorted(CONFIGS))
    ap.add_argument("--chunk-ctx", type=int, default=512 * 1024)
    ap.add_argument("--chunk-lat", type=int, default=128 * 1024,
                    help="T->D chunk: latent rows of one frame, C*W*4 bytes each (image: 16 rows; video: one frame)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--exclusive", action="store_true", help="N>1: E and D on GPUs of their own (1:N-2:1)")
    ap.add_argument("--t-per-gpu", type=int, default=1, help="DiT instances per GPU")
    ap.add_argument("--traffic", type=float, default=None,
                    help="dram bytes per launch of the dominant kernel from the committed ncu capture")
    ap.add_argument("--video-requests", type=int, default=1,
                    help="N=1 image run: timed C3 (video) requests in the line's `video` sub-record (0: skip)")
    ap.add_argument("--precision", default="bf16", choices=["bf16", "fp8", "mxfp8"],
                    help="the headline run's DiT precision (fp8: the R29 step mode; not a bf16 number)")
    ap.add_argument("--mxfp8-requests", type=int, default=5,
                    help="N=1 image run: timed requests of the MXFP8 step mode in the line's `mxfp8` sub-record (0: skip)")
    ap.add_argument("--fp8-requests", type=int, default=5,
                    help="N=1 image run: timed requests of the FP8 step mode in the line's `fp8` sub-record (0: skip)")
    ap.add_argument("--dit-steps", type=int, default=0,
                    help="Euler steps per request (0: the config's); for the few-step I2V / workload-shift runs")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if args.dit_steps:
        import dataclasses
        cfg = dataclasses.replace(cfg, steps=args.dit_steps)
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
