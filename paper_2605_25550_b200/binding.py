"""Thin ctypes binding of libdf (include/df.h): argument marshalling only.

Every computation runs inside libdf's CUDA kernels; this module converts Python
arguments (torch tensors -> device pointers, streams -> cudaStream_t) and raises
on a non-OK status.  There is no fallback: load() raises if libdf.so is missing.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libdf.so")

DF_OK, DF_AGAIN, DF_EMPTY = 0, 1, 2
DF_ERR_INVALID, DF_ERR_CAPACITY, DF_ERR_NOMEM, DF_ERR_DUPLICATE, DF_ERR_STATE = 10, 11, 12, 13, 14
DF_E, DF_T, DF_D = 0, 1, 2
DF_BF16, DF_FP32_VALIDATION, DF_FP8, DF_MXFP8 = 0, 1, 2, 3
DF_ASYNC, DF_SYNC, DF_PERMUTE, DF_HASH, DF_LATENT_BLOCKS = 0, 1, 2, 4, 8
DF_ALL_CHUNKS = 0xFFFFFFFF
DF_MAX_INST = 32


class DitCfgC(C.Structure):
    _fields_ = [("C", C.c_uint32), ("F", C.c_uint32), ("H", C.c_uint32), ("W", C.c_uint32),
                ("pt", C.c_uint32), ("ph", C.c_uint32), ("pw", C.c_uint32),
                ("d", C.c_uint32), ("heads", C.c_uint32), ("ffn", C.c_uint32), ("layers", C.c_uint32),
                ("d_txt", C.c_uint32), ("L_txt", C.c_uint32), ("freq_dim", C.c_uint32),
                ("vocab", C.c_uint32), ("enc_ffn", C.c_uint32), ("dec_width", C.c_uint32),
                ("eps", C.c_float), ("rope_theta", C.c_float), ("rope_axes", C.c_uint32 * 3),
                ("C_y", C.c_uint32), ("L_img", C.c_uint32), ("d_img", C.c_uint32)]


class InstC(C.Structure):
    _fields_ = [("device", C.c_int32), ("stage", C.c_int32), ("rank", C.c_int32)]


class GraphC(C.Structure):
    _fields_ = [("n_inst", C.c_uint32), ("inst", InstC * DF_MAX_INST), ("G", C.c_uint32),
                ("chunk_bytes", C.c_uint64 * 2), ("n_slots", C.c_uint32), ("handoff_mode", C.c_uint32),
                ("ring_capacity", C.c_uint32), ("precision", C.c_uint32), ("max_steps", C.c_uint32),
                ("weight_seed", C.c_uint64), ("jitter_p", C.c_float), ("jitter_delay_s", C.c_float),
                ("jitter_seed", C.c_uint64), ("dit", DitCfgC), ("rank", C.c_int32), ("world", C.c_int32),
                ("shm_name", C.c_char * 64), ("jitter_chunk", C.c_uint32)]


class ReqIdC(C.Structure):
    _fields_ = [("lo", C.c_uint64), ("hi", C.c_uint64)]


class RequestC(C.Structure):
    _fields_ = [("steps", C.c_uint32), ("shift", C.c_float), ("seed", C.c_uint64),
                ("token_ids", C.POINTER(C.c_int32)), ("out_host", C.c_void_p), ("out_bytes", C.c_uint64),
                ("user_tag", C.c_uint64), ("id", ReqIdC), ("guidance", C.c_float),
                ("neg_token_ids", C.POINTER(C.c_int32))]


class CompletionC(C.Structure):
    _fields_ = [("id", ReqIdC), ("status", C.c_int), ("user_tag", C.c_uint64), ("inst", C.c_int32 * 3),
                ("t_submit", C.c_double), ("t_start", C.c_double * 3), ("t_end", C.c_double * 3),
                ("t_done", C.c_double), ("stage_ms", C.c_float * 3), ("xfer_ms", C.c_float * 2),
                ("exposed_ms", C.c_float * 2), ("hash_src", C.c_uint64 * 2), ("hash_dst", C.c_uint64 * 2),
                ("out_view", C.c_void_p), ("out_view_bytes", C.c_uint64), ("overlap_ms", C.c_float * 2)]


class SchedCfgC(C.Structure):
    _fields_ = [("delta_s", C.c_float), ("U_high", C.c_float), ("U_low", C.c_float), ("Q_high", C.c_uint32),
                ("move_budget", C.c_int32), ("G", C.c_uint32)]


class SchedMetricsC(C.Structure):
    _fields_ = [("u", C.c_float * 3), ("q", C.c_uint32 * 3), ("d", C.c_float * 3)]


class SchedEventC(C.Structure):
    _fields_ = [("t", C.c_double), ("action", C.c_int32), ("stage", C.c_int32), ("g", C.c_uint32 * 3),
                ("m", SchedMetricsC), ("inst", C.c_int32), ("from_stage", C.c_int32), ("drain_ms", C.c_float),
                ("cold_start_ms", C.c_float)]


class HandoffDescC(C.Structure):
    _fields_ = [("src_inst", C.c_int32), ("dst_inst", C.c_int32), ("src", C.c_void_p), ("dst", C.c_void_p),
                ("bytes", C.c_uint64), ("chunk_bytes", C.c_uint64), ("flags", C.c_uint32),
                ("seq", C.c_uint64), ("edge", C.c_uint32)]


_lib = None

_SIGS = {
    "df_init": (C.c_int, [C.POINTER(GraphC), C.POINTER(C.c_void_p)]),
    "df_finalize": (C.c_int, [C.c_void_p]),
    "df_last_error": (C.c_char_p, [C.c_void_p]),
    "df_submit": (C.c_int, [C.c_void_p, C.POINTER(RequestC), C.POINTER(ReqIdC)]),
    "df_poll": (C.c_int, [C.c_void_p, C.POINTER(CompletionC), C.c_uint32, C.POINTER(C.c_uint32), C.c_int32]),
    "df_set_ratio": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32]),
    "df_dit_prepare": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.POINTER(C.c_float), C.c_uint32, C.c_void_p,
                                 C.POINTER(C.c_void_p)]),
    "df_dit_prepare_cfg": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_float, C.POINTER(C.c_float),
                                     C.c_uint32, C.c_void_p, C.POINTER(C.c_void_p)]),
    "df_dit_prepare_i2v": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_float,
                                     C.POINTER(C.c_float), C.c_uint32, C.c_void_p, C.POINTER(C.c_void_p)]),
    "df_dit_step": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_uint32, C.c_void_p, C.c_void_p, C.c_void_p]),
    "df_dit_layer": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p, C.c_void_p]),
    "df_cond_release": (C.c_int, [C.c_void_p, C.c_void_p]),
    "df_encode": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]),
    "df_decode": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]),
    "df_noise": (C.c_int, [C.c_void_p, C.c_int32, C.c_uint64, C.c_void_p, C.c_void_p]),
    "df_tokens": (C.c_int, [C.c_void_p, C.c_int32, C.c_uint64, C.c_void_p, C.c_void_p]),
    "df_image_cond": (C.c_int, [C.c_void_p, C.c_int32, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p]),
    "df_handoff": (C.c_int, [C.c_void_p, C.POINTER(HandoffDescC), C.c_void_p, C.POINTER(C.c_void_p)]),
    "df_handoff_wait": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint32, C.c_void_p]),
    "df_handoff_query": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(C.c_uint32), C.POINTER(C.c_uint64)]),
    "df_handoff_release": (C.c_int, [C.c_void_p, C.c_void_p]),
    "df_payload_hash": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64)]),
    "df_weight_bits": (C.c_int, [C.c_void_p, C.c_int32, C.c_uint32, C.c_void_p, C.c_uint64]),
    "df_op_gemm": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                             C.c_int32, C.c_void_p]),
    "df_op_attention": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32,
                                  C.c_int32, C.c_int32, C.c_int32, C.c_float, C.c_void_p]),
    "df_op_quant_e4m3": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p]),
    "df_op_gemm_e4m3": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32,
                                  C.c_int32, C.c_void_p, C.c_int32, C.c_void_p]),
    "df_op_qk_e4m3": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_float, C.c_void_p, C.c_void_p]),
    "df_op_attention_qf8": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32,
                                      C.c_int32, C.c_int32, C.c_float, C.c_void_p]),
    "df_op_attention_f8": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32,
                                     C.c_int32, C.c_int32, C.c_float, C.c_void_p, C.c_void_p, C.c_void_p]),
    "df_op_mx_quant_e4m3": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]),
    "df_op_gemm_mxf8": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32,
                                  C.c_int32, C.c_void_p, C.c_int32, C.c_void_p]),
    "df_op_rmsnorm_mod": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                                    C.c_float, C.c_void_p]),
    "df_launch_count": (C.c_uint64, [C.c_void_p]),
    "df_chunk_plan": (C.c_int, [C.POINTER(GraphC), C.c_uint32, C.c_uint64, C.POINTER(C.c_uint32),
                                C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                                C.POINTER(C.c_uint64), C.c_uint32]),
    "df_plan_ratio": (C.c_int, [C.c_uint32, C.POINTER(C.c_double), C.POINTER(C.c_uint32), C.c_int32,
                                C.POINTER(C.c_uint32)]),
    "df_sched_react": (C.c_int, [C.POINTER(SchedCfgC), C.POINTER(SchedMetricsC), C.POINTER(SchedMetricsC),
                                 C.POINTER(C.c_uint32), C.POINTER(C.c_int32)]),
    "df_sched_changed": (C.c_int32, [C.POINTER(C.c_uint32), C.c_uint32]),
    "df_sched_start": (C.c_int, [C.c_void_p, C.POINTER(SchedCfgC)]),
    "df_sched_stop": (C.c_int, [C.c_void_p]),
    "df_sched_log": (C.c_int, [C.c_void_p, C.POINTER(SchedEventC), C.c_uint32, C.POINTER(C.c_uint32)]),
    "df_ring_selftest": (C.c_int, [C.c_char_p, C.c_int32, C.c_uint64, C.POINTER(C.c_uint64), C.POINTER(C.c_int32)]),
    "df_profile": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32]),
    "df_kernel_stats": (C.c_int, [C.c_void_p, C.c_uint32, C.POINTER(C.c_uint64), C.POINTER(C.c_double),
                                  C.POINTER(C.c_double), C.POINTER(C.c_double)]),
}

EXPORTS = tuple(_SIGS)


def load(path: str = LIB_PATH):
    """Load libdf.so (no fallback: raises if it is missing)."""
    global _lib
    if _lib is None:
        if not os.path.exists(path):
            raise RuntimeError(f"libdf.so not built at {path}: run `python -m paper_2605_25550_b200.build`")
        lib = C.CDLL(path)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


class DFError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"libdf status {status}: {msg}")
        self.status = status


def dit_cfg_c(cfg) -> DitCfgC:
    """synth.configs.DitCfg -> df_dit_cfg."""
    c = DitCfgC()
    for k in ("C", "F", "H", "W", "pt", "ph", "pw", "d", "heads", "ffn", "layers", "d_txt", "L_txt", "freq_dim",
              "vocab", "dec_width", "C_y", "L_img", "d_img"):
        setattr(c, k, int(getattr(cfg, k)))
    c.enc_ffn = int(cfg.f_e)
    c.eps = float(cfg.eps)
    c.rope_theta = float(cfg.rope_theta)
    for i, a in enumerate(cfg.rope_axes):
        c.rope_axes[i] = int(a)
    return c


def make_graph(cfg, instances, precision=DF_BF16, weight_seed=0, chunk_bytes=(0, 0), n_slots=2,
               handoff_mode=DF_ASYNC | DF_HASH, ring_capacity=256, max_steps=None, jitter=(0.0, 0.0, 0), G=0,
               rank=0, world=1, shm_name="", jitter_chunk=0):
    """instances: list of (device, stage) or (device, stage, rank)."""
    g = GraphC()
    g.n_inst = len(instances)
    for i, ins in enumerate(instances):
        g.inst[i].device = int(ins[0])
        g.inst[i].stage = int(ins[1])
        g.inst[i].rank = int(ins[2]) if len(ins) > 2 else 0
    g.rank, g.world = int(rank), int(world)
    g.shm_name = shm_name.encode()[:63]
    g.G = int(G)
    g.chunk_bytes[0], g.chunk_bytes[1] = int(chunk_bytes[0]), int(chunk_bytes[1])
    g.n_slots = int(n_slots)
    g.handoff_mode = int(handoff_mode)
    g.ring_capacity = int(ring_capacity)
    g.precision = int(precision)
    g.max_steps = int(max_steps if max_steps is not None else max(cfg.steps, 64))
    g.weight_seed = int(weight_seed)
    g.jitter_p, g.jitter_delay_s, g.jitter_seed = float(jitter[0]), float(jitter[1]), int(jitter[2])
    g.jitter_chunk = int(jitter_chunk)
    g.dit = dit_cfg_c(cfg)
    return g


def sched_cfg(delta_s=2.0, U_high=0.8, U_low=0.2, Q_high=5, move_budget=-1, G=0) -> SchedCfgC:
    """Alg. 1 defaults."""
    return SchedCfgC(float(delta_s), float(U_high), float(U_low), int(Q_high), int(move_budget), int(G))


def plan_ratio(G, T, cur=None, budget=-1):
    lib = load()
    Tc = (C.c_double * 3)(*T)
    out = (C.c_uint32 * 3)()
    curc = (C.c_uint32 * 3)(*cur) if cur is not None else None
    st = lib.df_plan_ratio(int(G), Tc, curc, int(budget), out)
    if st != DF_OK:
        raise DFError(st, "df_plan_ratio")
    return tuple(out)


def sched_react(cfg, now, prev, g):
    lib = load()
    def mk(m):
        if m is None:
            return None
        u, q, d = m
        return C.byref(SchedMetricsC((C.c_float * 3)(*u), (C.c_uint32 * 3)(*q), (C.c_float * 3)(*d)))
    out = (C.c_int32 * 3)()
    st = lib.df_sched_react(C.byref(cfg), mk(now), mk(prev), (C.c_uint32 * 3)(*g), out)
    if st != DF_OK:
        raise DFError(st, "df_sched_react")
    return tuple(out)


def chunk_plan(graph, edge, nbytes, max_pieces=64):
    """The pipeline edge's chunk plan (host logic): [(off, width, height, pitch)]."""
    lib = load()
    n = C.c_uint32()
    arrs = [(C.c_uint64 * max_pieces)() for _ in range(4)]
    st = lib.df_chunk_plan(C.byref(graph), int(edge), int(nbytes), C.byref(n), *arrs, max_pieces)
    if st != DF_OK:
        raise DFError(st, "df_chunk_plan")
    return [tuple(int(a[k]) for a in arrs) for k in range(min(n.value, max_pieces))]


def sched_changed(keys):
    lib = load()
    arr = (C.c_uint32 * max(1, len(keys)))(*keys)
    return bool(lib.df_sched_changed(arr, len(keys)))


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(s):
    if s is None:
        import torch
        s = torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


class Context:
    """Owns one df_ctx.  Methods mirror the C ABI names."""

    def __init__(self, graph: GraphC):
        self.lib = load()
        self.h = C.c_void_p()
        st = self.lib.df_init(C.byref(graph), C.byref(self.h))
        if st != DF_OK:
            raise DFError(st, self.lib.df_last_error(None).decode())
        self.graph = graph

    def _ck(self, st, ok=(DF_OK,)):
        if st not in ok:
            raise DFError(st, self.lib.df_last_error(self.h).decode())
        return st

    def close(self):
        if self.h:
            self.lib.df_finalize(self.h)
            self.h = C.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # ---- serving
    def submit(self, steps, shift, seed, out_host=None, token_ids=None, user_tag=0, req_id=None, guidance=1.0,
               neg_token_ids=None):
        r = RequestC()
        r.steps, r.shift, r.seed, r.user_tag = int(steps), float(shift), int(seed), int(user_tag)
        r.guidance = float(guidance)
        if neg_token_ids is not None:
            self._nids = (C.c_int32 * len(neg_token_ids))(*[int(x) for x in neg_token_ids])
            r.neg_token_ids = C.cast(self._nids, C.POINTER(C.c_int32))
        if token_ids is not None:
            self._ids = (C.c_int32 * len(token_ids))(*[int(x) for x in token_ids])
            r.token_ids = C.cast(self._ids, C.POINTER(C.c_int32))
        if out_host is not None:
            r.out_host = C.c_void_p(out_host.ctypes.data if hasattr(out_host, "ctypes") else out_host.data_ptr())
            r.out_bytes = out_host.nbytes if hasattr(out_host, "nbytes") else out_host.numel() * out_host.element_size()
        if req_id is not None:
            r.id.lo, r.id.hi = req_id
        rid = ReqIdC()
        st = self.lib.df_submit(self.h, C.byref(r), C.byref(rid))
        self._ck(st, ok=(DF_OK, DF_AGAIN))
        return st, (rid.lo, rid.hi)

    def poll(self, max_n=64, timeout_ms=100):
        arr = (CompletionC * max_n)()
        n = C.c_uint32()
        st = self.lib.df_poll(self.h, arr, max_n, C.byref(n), int(timeout_ms))
        self._ck(st, ok=(DF_OK, DF_EMPTY))
        return [arr[i] for i in range(n.value)]

    def set_ratio(self, gE, gT, gD):
        return self._ck(self.lib.df_set_ratio(self.h, gE, gT, gD), ok=(DF_OK, DF_ERR_CAPACITY))

    # ---- low level
    def dit_prepare(self, t_inst, ctx_dev, sigmas, stream=None):
        sig = (C.c_float * len(sigmas))(*[float(s) for s in sigmas])
        out = C.c_void_p()
        self._ck(self.lib.df_dit_prepare(self.h, t_inst, _ptr(ctx_dev), sig, len(sigmas) - 1, _stream(stream),
                                         C.byref(out)))
        return out

    def dit_prepare_cfg(self, t_inst, ctx_dev, ctx_neg_dev, guidance, sigmas, stream=None):
        sig = (C.c_float * len(sigmas))(*[float(s) for s in sigmas])
        out = C.c_void_p()
        self._ck(self.lib.df_dit_prepare_cfg(self.h, t_inst, _ptr(ctx_dev), _ptr(ctx_neg_dev), float(guidance), sig,
                                             len(sigmas) - 1, _stream(stream), C.byref(out)))
        return out

    def dit_prepare_i2v(self, t_inst, ctx_dev, clip_dev, y_dev, sigmas, ctx_neg_dev=None, guidance=1.0, stream=None):
        sig = (C.c_float * len(sigmas))(*[float(s) for s in sigmas])
        out = C.c_void_p()
        self._ck(self.lib.df_dit_prepare_i2v(self.h, t_inst, _ptr(ctx_dev), _ptr(clip_dev), _ptr(y_dev),
                                             _ptr(ctx_neg_dev), float(guidance), sig, len(sigmas) - 1,
                                             _stream(stream), C.byref(out)))
        return out

    def dit_step(self, t_inst, cond, i, x_dev, v_dev=None, stream=None):
        self._ck(self.lib.df_dit_step(self.h, t_inst, cond, i, _ptr(x_dev), _ptr(v_dev), _stream(stream)))

    def dit_layer(self, t_inst, cond, i, l, r_dev, stream=None):
        self._ck(self.lib.df_dit_layer(self.h, t_inst, cond, i, l, _ptr(r_dev), _stream(stream)))

    def cond_release(self, cond):
        self._ck(self.lib.df_cond_release(self.h, cond))

    def encode(self, e_inst, ids_dev, ctx_dev, stream=None):
        self._ck(self.lib.df_encode(self.h, e_inst, _ptr(ids_dev), _ptr(ctx_dev), _stream(stream)))

    def decode(self, d_inst, x_dev, out_dev, stream=None):
        self._ck(self.lib.df_decode(self.h, d_inst, _ptr(x_dev), _ptr(out_dev), _stream(stream)))

    def noise(self, inst, seed, x_dev, stream=None):
        self._ck(self.lib.df_noise(self.h, inst, seed, _ptr(x_dev), _stream(stream)))

    def tokens(self, inst, seed, ids_dev, stream=None):
        self._ck(self.lib.df_tokens(self.h, inst, seed, _ptr(ids_dev), _stream(stream)))

    def image_cond(self, inst, seed, clip_dev, y_dev, stream=None):
        self._ck(self.lib.df_image_cond(self.h, inst, seed, _ptr(clip_dev), _ptr(y_dev), _stream(stream)))

    def handoff(self, src_inst, dst_inst, src, dst, nbytes, chunk_bytes, flags=0, seq=0, edge=0, stream=None):
        d = HandoffDescC(src_inst, dst_inst, C.c_void_p(src.data_ptr()), C.c_void_p(dst.data_ptr()), int(nbytes),
                         int(chunk_bytes), int(flags), int(seq), int(edge))
        x = C.c_void_p()
        self._ck(self.lib.df_handoff(self.h, C.byref(d), _stream(stream), C.byref(x)))
        return x

    def handoff_wait(self, x, chunk=DF_ALL_CHUNKS, stream=None):
        self._ck(self.lib.df_handoff_wait(self.h, x, chunk, _stream(stream)))

    def handoff_query(self, x):
        n = C.c_uint32()
        h = (C.c_uint64 * 2)()
        self._ck(self.lib.df_handoff_query(self.h, x, C.byref(n), h))
        return n.value, (h[0], h[1])

    def handoff_release(self, x):
        self._ck(self.lib.df_handoff_release(self.h, x))

    def payload_hash(self, inst, buf_dev, nbytes):
        h = C.c_uint64()
        self._ck(self.lib.df_payload_hash(self.h, inst, _ptr(buf_dev), int(nbytes), C.byref(h)))
        return h.value

    def weight_bits(self, inst, tensor_id, n):
        import numpy as np
        out = np.empty(n, dtype=np.uint16)
        self._ck(self.lib.df_weight_bits(self.h, inst, int(tensor_id), out.ctypes.data_as(C.c_void_p), int(n)))
        return out

    def op_gemm(self, A, W, out, tc=1, stream=None):
        M, K = A.shape
        N = W.shape[0]
        self._ck(self.lib.df_op_gemm(self.h, _ptr(A), _ptr(W), _ptr(out), M, N, K, int(tc), _stream(stream)))

    def op_quant_e4m3(self, x, q, scale, stream=None):
        """x: bf16 (any shape, contiguous); q: uint8 of x.numel(); scale: fp32 [1] (device)."""
        self._ck(self.lib.df_op_quant_e4m3(self.h, _ptr(x), int(x.numel()), _ptr(q), _ptr(scale), _stream(stream)))

    def op_gemm_e4m3(self, qa, qb, sa, sb, out, stream=None):
        """qa uint8 [M,K], qb uint8 [N,K], sa/sb fp32 [1] (device), out fp32 or bf16 [M,N]."""
        M, K = qa.shape
        N = qb.shape[0]
        out_f32 = int(str(out.dtype) == "torch.float32")
        self._ck(self.lib.df_op_gemm_e4m3(self.h, _ptr(qa), _ptr(qb), _ptr(sa), _ptr(sb), M, N, K, _ptr(out), out_f32,
                                          _stream(stream)))

    def op_qk_e4m3(self, x, inv, q, stream=None):
        """x bf16 (any shape, contiguous, numel % 8 == 0); q uint8 of x.numel()."""
        self._ck(self.lib.df_op_qk_e4m3(self.h, _ptr(x), int(x.numel()), float(inv), _ptr(q), _stream(stream)))

    def op_attention_qf8(self, Q8, K8, V, O, H, Nq, Nk, scale, stream=None):
        self._ck(self.lib.df_op_attention_qf8(self.h, _ptr(Q8), _ptr(K8), _ptr(V), _ptr(O), H, Nq, Nk, float(scale),
                                              _stream(stream)))

    def op_attention_f8(self, Q8, K8, V, O, H, Nq, Nk, scale, v8t, vscale, stream=None):
        self._ck(self.lib.df_op_attention_f8(self.h, _ptr(Q8), _ptr(K8), _ptr(V), _ptr(O), H, Nq, Nk, float(scale),
                                             _ptr(v8t), _ptr(vscale), _stream(stream)))

    def op_mx_quant_e4m3(self, x, q, sf, stream=None):
        """x bf16 [M, K] (K % 128 == 0); q uint8 [M, K]; sf uint8 of (K/128) * ceil(M/128) * 512 bytes."""
        M, K = x.shape
        self._ck(self.lib.df_op_mx_quant_e4m3(self.h, _ptr(x), M, K, _ptr(q), _ptr(sf), _stream(stream)))

    def op_gemm_mxf8(self, qa, sa, qb, sb, out, stream=None):
        """qa uint8 [M,K], qb uint8 [N,K], sa/sb tiled E8M0 scale bytes, out fp32 or bf16 [M,N]."""
        M, K = qa.shape
        N = qb.shape[0]
        out_f32 = int(str(out.dtype) == "torch.float32")
        self._ck(self.lib.df_op_gemm_mxf8(self.h, _ptr(qa), _ptr(sa), _ptr(qb), _ptr(sb), M, N, K, _ptr(out), out_f32,
                                          _stream(stream)))

    def op_attention(self, Q, K, V, O, H, Nq, Nk, dh, dh_pad, scale, stream=None):
        self._ck(self.lib.df_op_attention(self.h, _ptr(Q), _ptr(K), _ptr(V), _ptr(O), H, Nq, Nk, dh, dh_pad,
                                          float(scale), _stream(stream)))

    def op_rmsnorm_mod(self, x, out, shift, scale, eps, stream=None):
        M, d = x.shape
        self._ck(self.lib.df_op_rmsnorm_mod(self.h, _ptr(x), _ptr(out), M, d, _ptr(shift), _ptr(scale), float(eps),
                                            _stream(stream)))

    KINDS = ("qkv", "attn_self", "o_proj", "rmsnorm", "cross_q", "attn_cross", "cross_o", "mlp_up", "mlp_down",
             "head_euler", "patch_embed")

    def profile(self, enable=True, reset=True):
        self._ck(self.lib.df_profile(self.h, int(enable), int(reset)))

    def kernel_stats(self):
        out = {}
        for k, name in enumerate(self.KINDS):
            n, ms, fl, by = C.c_uint64(), C.c_double(), C.c_double(), C.c_double()
            self._ck(self.lib.df_kernel_stats(self.h, k, C.byref(n), C.byref(ms), C.byref(fl), C.byref(by)))
            out[name] = {"launches": n.value, "ms": ms.value, "flops": fl.value, "bytes": by.value}
        return out

    def sched_start(self, cfg):
        self._ck(self.lib.df_sched_start(self.h, C.byref(cfg)))

    def sched_stop(self):
        self._ck(self.lib.df_sched_stop(self.h))

    def sched_log(self):
        n = C.c_uint32()
        self._ck(self.lib.df_sched_log(self.h, None, 0, C.byref(n)))
        arr = (SchedEventC * max(1, n.value))()
        self._ck(self.lib.df_sched_log(self.h, arr, n.value, C.byref(n)))
        return [arr[i] for i in range(n.value)]

    def launch_count(self):
        return int(self.lib.df_launch_count(self.h))
