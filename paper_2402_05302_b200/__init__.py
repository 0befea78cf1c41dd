"""B200-native hot path of Cannikin (arXiv 2402.05302): thin Python binding of libcannikin.so.

Argument marshalling only -- every step of the path runs in the CUDA library (device kernels) or
its C++ host solvers.  There is no fallback: if the library is missing this import fails.

Entry points mirror include/cannikin.h:
    Context(...)                      cannikin_init / cannikin_destroy
    Context.alloc_bucket / free_bucket
    Context.weighted_allreduce        Eq. 9 + fused |g_i|^2, |g|^2
    weighted_allreduce_group          the same for every rank of an in-process group, one launch
    Context.weighted_allreduce_nccl   the same through NCCL reduce-scatter / all-gather (K4)
    Context.gns_stats                 finalise the norm statistics
    Context.weighted_sum_local        emulated ranks on one GPU
    gns_estimate                      Eq. 10 + Theorem 1
    opt_split                         OptPerf split
    warmup_split, node_time           Eq. 8; Eq. 5-7 frozen evaluation
Torch-tensor conveniences live in ``paper_2402_05302_b200.torch_api``.
"""
from __future__ import annotations

import ctypes
import os

__all__ = [
    "CannikinError", "Context", "F32", "BF16", "ACCUMULATE", "ROUND_PAPER", "lib", "lib_path",
    "get_unique_id", "gns_estimate", "opt_split", "node_time", "warmup_split", "MAX_WORLD",
    "weighted_allreduce_group",
    "MAX_EMULATED",
]

F32, BF16 = 0, 1
ACCUMULATE = 1
LOCAL_LDG = 2
LOCAL_TMA = 4
LOCAL_CHAIN = 8
ROUND_PAPER = 1
GNS_G_NONPOSITIVE = 1
MAX_WORLD = 8
MAX_EMULATED = 16
MAX_GNS = 64

_STATUS = {0: "OK", 1: "INVALID", 2: "DOMAIN", 3: "INFEASIBLE", 4: "SINGULAR", 5: "CUDA", 6: "NCCL",
           7: "UNSUPPORTED"}

_HERE = os.path.dirname(os.path.abspath(__file__))


def lib_path() -> str:
    # CANNIKIN_LIB: an alternative build of the same library (tools' build-time A/B runs only)
    return os.environ.get("CANNIKIN_LIB") or os.path.join(_HERE, "libcannikin.so")


class CannikinError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"cannikin {_STATUS.get(status, status)}: {msg}")
        self.status = status
        self.name = _STATUS.get(status, str(status))


class _GnsResult(ctypes.Structure):
    _fields_ = [("G2", ctypes.c_double), ("trS", ctypes.c_double), ("B_noise", ctypes.c_double),
                ("Gi", ctypes.c_double * MAX_GNS), ("Si", ctypes.c_double * MAX_GNS),
                ("wG", ctypes.c_double * MAX_GNS), ("wS", ctypes.c_double * MAX_GNS),
                ("n", ctypes.c_int), ("flags", ctypes.c_uint)]


class _NodeModel(ctypes.Structure):
    _fields_ = [("q", ctypes.c_double), ("s", ctypes.c_double), ("k", ctypes.c_double),
                ("m", ctypes.c_double)]


class _CommModel(ctypes.Structure):
    _fields_ = [("gamma", ctypes.c_double), ("t_o", ctypes.c_double), ("t_u", ctypes.c_double)]


class _GnsEma(ctypes.Structure):
    _fields_ = [("G2", ctypes.c_double), ("trS", ctypes.c_double), ("decay", ctypes.c_double),
                ("count", ctypes.c_int), ("B_noise", ctypes.c_double)]


_LIB = None

# Every symbol include/cannikin.h declares, with (restype, argtypes).
_P, _D, _I, _U, _Z, _L = (ctypes.c_void_p, ctypes.c_double, ctypes.c_int, ctypes.c_uint,
                          ctypes.c_size_t, ctypes.c_int64)
_DP, _LP, _IP = (ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64),
                 ctypes.POINTER(ctypes.c_int))
SIGNATURES = {
    "cannikin_last_error": (ctypes.c_char_p, []),
    "cannikin_version": (_I, []),
    "cannikin_get_unique_id": (_I, [_P]),
    "cannikin_init": (_I, [ctypes.POINTER(_P), _I, _I, _P, _I, _Z, _I, _U]),
    "cannikin_destroy": (_I, [_P]),
    "cannikin_init_group_local": (_I, [ctypes.POINTER(_P), _I, _I, _Z, _I, _U]),
    "cannikin_alloc_bucket": (_I, [_P, _Z, ctypes.POINTER(_P)]),
    "cannikin_free_bucket": (_I, [_P, _P]),
    "cannikin_weighted_allreduce": (_I, [_P, _P, _Z, _I, _D, _P]),
    "cannikin_weighted_allreduce_group": (_I, [ctypes.POINTER(_P), _I, ctypes.POINTER(_P), _Z, _I,
                                               _DP, _P]),
    "cannikin_weighted_allreduce_nvls": (_I, [_P, _P, _P, _Z, _I, _D, _P]),
    "cannikin_weighted_allreduce_nccl": (_I, [_P, _P, _Z, _I, _D, _P]),
    "cannikin_gns_stats": (_I, [_P, _P, _DP, _DP]),
    "cannikin_gns_stats_async": (_I, [_P, _P, _P]),
    "cannikin_gns_stats_bucket": (_I, [_P, _P, _Z, _I, _L, _P, _DP, _DP]),
    "cannikin_device_status": (_I, [_P]),
    "cannikin_weighted_sum_local": (_I, [_P, ctypes.POINTER(_P), _I, _DP, _P, _Z, _I, _P, _P, _U, _P]),
    "cannikin_ddp_allreduce_mean": (_I, [_P, _P, _Z, _I, _P]),
    "cannikin_last_launch_count": (_I, [_P]),
    "cannikin_last_variant": (ctypes.c_char_p, [_P]),
    "cannikin_emulate_compute": (_I, [_D, _P]),
    "cannikin_probe_a2a_write": (_I, [_P, _Z, _I, _I, _P]),
    "cannikin_probe_stream_pattern": (_I, [ctypes.POINTER(_P), _I, _P, _Z, _I, _P]),
    "cannikin_green_partitions": (_I, [_I, _I, _IP, ctypes.POINTER(_P), ctypes.POINTER(_P), _IP]),
    "cannikin_green_destroy": (_I, [_P]),
    "cannikin_trace": (_I, [_P, ctypes.POINTER(ctypes.c_uint64), _I, _IP]),
    "cannikin_gns_estimate": (_I, [_DP, _D, _LP, _I, ctypes.POINTER(_GnsResult)]),
    "cannikin_gns_estimate_corrected": (_I, [_DP, _D, _LP, _I, ctypes.POINTER(_GnsResult)]),
    "cannikin_node_time": (_D, [ctypes.POINTER(_NodeModel), ctypes.POINTER(_CommModel), _D]),
    "cannikin_opt_split": (_I, [ctypes.POINTER(_NodeModel), _I, ctypes.POINTER(_CommModel), _L, _LP,
                                _LP, _U, _LP, _DP, _DP, _IP]),
    "cannikin_warmup_split": (_I, [_DP, _I, _L, _DP, _LP]),
    "cannikin_fit_linear": (_I, [_DP, _DP, _I, _DP, _DP]),
    "cannikin_ivw": (_I, [_DP, _DP, _I, _DP]),
    "cannikin_analyzer_create": (_I, [_I, ctypes.POINTER(_P)]),
    "cannikin_analyzer_destroy": (_I, [_P]),
    "cannikin_analyzer_observe": (_I, [_P, _I, _L, _L, _D, _D, _D, _D, _D]),
    "cannikin_analyzer_models": (_I, [_P, ctypes.POINTER(_NodeModel), ctypes.POINTER(_CommModel)]),
    "cannikin_analyzer_plan": (_I, [_P, _L, _LP, _LP, _DP, _IP]),
    "cannikin_gns_ema_update": (_I, [ctypes.POINTER(_GnsEma), _D, _D]),
    "cannikin_efficiency": (_D, [_L, _L, _D]),
    "cannikin_choose_batch": (_I, [ctypes.POINTER(_NodeModel), _I, ctypes.POINTER(_CommModel), _LP,
                                   _I, _L, _D, _LP, _DP, _DP]),
    "cannikin_analyzer_choose_batch": (_I, [_P, _LP, _I, _L, _D, _LP, _LP, _DP, _IP]),
    "cannikin_control_step": (_I, [_DP, _LP, _I, ctypes.POINTER(_GnsEma), ctypes.POINTER(_NodeModel),
                                   ctypes.POINTER(_CommModel), _L, ctypes.POINTER(_GnsResult), _LP,
                                   _DP]),
}


def lib() -> ctypes.CDLL:
    """Load libcannikin.so (built in-tree by paper_2402_05302_b200.build).  No fallback."""
    global _LIB
    if _LIB is None:
        path = lib_path()
        if not os.path.exists(path):
            raise ImportError(f"{path} is missing: run `python -m paper_2402_05302_b200.build` "
                              "(there is no CPU fallback)")
        L = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype, f.argtypes = res, args
        _LIB = L
    return _LIB


def _check(status: int):
    if status != 0:
        raise CannikinError(status, lib().cannikin_last_error().decode())


def _dbl(xs):
    return (ctypes.c_double * len(xs))(*[float(x) for x in xs])


def _i64(xs):
    return (ctypes.c_int64 * len(xs))(*[int(x) for x in xs])


def _stream(s) -> int | None:
    if s is None:
        return None
    if isinstance(s, int):
        return s
    return int(getattr(s, "cuda_stream"))


# ----------------------------------------------------------------------------- device context
INIT_CHECK_RATIOS = 1  # cannikin.h CANNIKIN_INIT_CHECK_RATIOS
INIT_GATED_ENTRY = 2   # cannikin.h CANNIKIN_INIT_GATED_ENTRY


class Context:
    """A cannikin_ctx: one per (process, GPU).  world > 1 is collective (see cannikin_init)."""

    def __init__(self, rank: int = 0, world: int = 1, unique_id: bytes | None = None,
                 device: int = 0, heap_bytes: int = 0, grid: int = 0,
                 check_ratios: bool = False, gated: bool = False):
        L = lib()
        h = ctypes.c_void_p()
        uid = None
        if unique_id is not None:
            assert len(unique_id) == 128
            uid = ctypes.create_string_buffer(bytes(unique_id), 128)
        flags = (INIT_CHECK_RATIOS if check_ratios else 0) | (INIT_GATED_ENTRY if gated else 0)
        _check(L.cannikin_init(ctypes.byref(h), rank, world, uid, device, heap_bytes, grid, flags))
        self._h = h
        self.rank, self.world, self.device = rank, world, device

    @classmethod
    def group_local(cls, world: int, device: int = 0, heap_bytes: int = 0, grid: int = 0,
                    check_ratios: bool = False) -> list:
        """cannikin_init_group_local: `world` ranks on ONE device in this process (their
        reductions must be issued concurrently, one stream per rank)."""
        hs = (_P * world)()
        flags = INIT_CHECK_RATIOS if check_ratios else 0
        _check(lib().cannikin_init_group_local(hs, world, device, heap_bytes, grid, flags))
        out = []
        for k in range(world):
            c = cls.__new__(cls)
            c._h = ctypes.c_void_p(hs[k])
            c.rank, c.world, c.device = k, world, device
            out.append(c)
        return out

    def close(self):
        if getattr(self, "_h", None):
            _check(lib().cannikin_destroy(self._h))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def alloc_bucket(self, nbytes: int) -> int:
        p = ctypes.c_void_p()
        _check(lib().cannikin_alloc_bucket(self._h, nbytes, ctypes.byref(p)))
        return int(p.value)

    def free_bucket(self, ptr: int):
        _check(lib().cannikin_free_bucket(self._h, ptr))

    def weighted_allreduce(self, ptr: int, n: int, dtype: int, r_i: float, stream=None):
        _check(lib().cannikin_weighted_allreduce(self._h, ptr, n, dtype, r_i, _stream(stream)))

    def weighted_allreduce_nccl(self, ptr: int, n: int, dtype: int, r_i: float, stream=None):
        _check(lib().cannikin_weighted_allreduce_nccl(self._h, ptr, n, dtype, r_i, _stream(stream)))

    def weighted_allreduce_nvls(self, ptr: int, mc_ptr: int, n: int, dtype: int, r_i: float,
                                stream=None):
        _check(lib().cannikin_weighted_allreduce_nvls(self._h, ptr, mc_ptr, n, dtype, r_i,
                                                      _stream(stream)))

    def gns_stats(self, stream=None):
        out = (ctypes.c_double * self.world)()
        g = ctypes.c_double()
        _check(lib().cannikin_gns_stats(self._h, _stream(stream), out, ctypes.byref(g)))
        return list(out), g.value

    def gns_stats_bucket(self, ptr: int, n: int, dtype: int, b_i: int, stream=None):
        """Out-of-place statistics of one bucket (cannikin_gns_stats_bucket): (|g_j|^2 for every
        rank j, |g|^2) with g = sum_j (b_j / B) g_j; the bucket is not modified.  Collective."""
        out = (ctypes.c_double * self.world)()
        g = ctypes.c_double()
        _check(lib().cannikin_gns_stats_bucket(self._h, ptr, n, dtype, int(b_i), _stream(stream),
                                               out, ctypes.byref(g)))
        return list(out), g.value

    def gns_stats_async(self, d_out: int, stream=None):
        _check(lib().cannikin_gns_stats_async(self._h, d_out, _stream(stream)))

    def device_status(self):
        """Raise CannikinError for a condition the reduction kernels recorded (DOMAIN: shares not
        summing to 1 under check_ratios -- cleared by this call)."""
        _check(lib().cannikin_device_status(self._h))

    def weighted_sum_local(self, in_ptrs, r, out_ptr: int, n: int, dtype: int, d_local_sq: int,
                           d_global_sq: int, accumulate: bool = False, stream=None,
                           variant: str | None = None, chain: bool = False):
        """variant: None (library default), "ldg" or "tma": same per-element arithmetic (identical
        output bits); the fp64 norm partials differ only in summation grouping.  chain: the inputs
        are not written by the kernel enqueued just before (CANNIKIN_LOCAL_CHAIN)."""
        arr = (ctypes.c_void_p * len(in_ptrs))(*in_ptrs)
        flags = (ACCUMULATE if accumulate else 0) | {None: 0, "ldg": LOCAL_LDG,
                                                     "tma": LOCAL_TMA}[variant]
        flags |= LOCAL_CHAIN if chain else 0
        _check(lib().cannikin_weighted_sum_local(self._h, arr, len(in_ptrs), _dbl(r), out_ptr, n,
                                                 dtype, d_local_sq, d_global_sq, flags,
                                                 _stream(stream)))

    def ddp_allreduce_mean(self, ptr: int, n: int, dtype: int, stream=None):
        _check(lib().cannikin_ddp_allreduce_mean(self._h, ptr, n, dtype, _stream(stream)))

    def trace(self, max_ctas: int = 2048):
        """Per-CTA timeline (ns) of the last two-shot kernel: list of [start, entry, data, exit,
        end] (end only set on the last CTA to finish)."""
        buf = (ctypes.c_uint64 * (5 * max_ctas))()
        n = ctypes.c_int()
        _check(lib().cannikin_trace(self._h, buf, max_ctas, ctypes.byref(n)))
        return [list(buf[5 * i:5 * i + 5]) for i in range(n.value)]

    def last_launch_count(self) -> int:
        return int(lib().cannikin_last_launch_count(self._h))

    def last_variant(self) -> str:
        return lib().cannikin_last_variant(self._h).decode()

    def probe_a2a_write(self, bytes_per_peer: int, repeat: int = 1, ctas_per_sm: int = 2,
                        stream=None):
        """cannikin_probe_a2a_write (bench utility, COLLECTIVE): all-to-all peer writes."""
        _check(lib().cannikin_probe_a2a_write(self._h, int(bytes_per_peer), int(repeat),
                                              int(ctas_per_sm), _stream(stream)))


def weighted_allreduce_group(ctxs, ptrs, n: int, dtype: int, r, stream=None):
    """cannikin_weighted_allreduce_group: every rank of an in-process group (Context.group_local,
    in rank order) reduced by ONE kernel launch on `stream`."""
    w = len(ctxs)
    hs = (_P * w)(*[c._h.value for c in ctxs])
    ps = (_P * w)(*ptrs)
    _check(lib().cannikin_weighted_allreduce_group(hs, w, ps, n, dtype, _dbl(r), _stream(stream)))


class GreenPartitions:
    """cannikin_green_partitions (bench utility): disjoint SM partitions of one GPU, one stream
    each.  `streams` are raw cudaStream_t handles (use torch.cuda.ExternalStream), `sms` the SMs
    each partition received."""

    def __init__(self, sm_counts, device: int = 0):
        n = len(sm_counts)
        h = _P()
        st = (_P * n)()
        got = (ctypes.c_int * n)()
        _check(lib().cannikin_green_partitions(device, n, (ctypes.c_int * n)(*sm_counts),
                                               ctypes.byref(h), st, got))
        self._h = h
        self.streams = [int(st[i]) for i in range(n)]
        self.sms = list(got)

    def close(self):
        if self._h:
            _check(lib().cannikin_green_destroy(self._h))
            self._h = None


def probe_stream_pattern(in_ptrs, out_ptr: int, nbytes: int, ctas_per_sm: int = 4, stream=None):
    """cannikin_probe_stream_pattern (bench utility): the bare n:1 memory pattern of K2."""
    n = len(in_ptrs)
    _check(lib().cannikin_probe_stream_pattern((_P * n)(*in_ptrs), n, out_ptr, int(nbytes),
                                               int(ctas_per_sm), _stream(stream)))


def emulate_compute(seconds: float, stream=None):
    """Bench utility: synthetic compute of `seconds` device time on `stream` (K7)."""
    _check(lib().cannikin_emulate_compute(float(seconds), _stream(stream)))


def get_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().cannikin_get_unique_id(buf))
    return buf.raw


# ----------------------------------------------------------------------------- host solvers
def gns_estimate(local_sq, global_sq: float, b, corrected: bool = False) -> dict:
    """Theorem 1 as printed (default), or the corrected-covariance variant (corrected=True)."""
    n = len(b)
    res = _GnsResult()
    fn = lib().cannikin_gns_estimate_corrected if corrected else lib().cannikin_gns_estimate
    _check(fn(_dbl(local_sq), float(global_sq), _i64(b), n, ctypes.byref(res)))
    return {"G2": res.G2, "trS": res.trS, "B_noise": res.B_noise, "Gi": list(res.Gi[:n]),
            "Si": list(res.Si[:n]), "wG": list(res.wG[:n]), "wS": list(res.wS[:n]),
            "flags": res.flags}


def _models(nodes, comm):
    arr = (_NodeModel * len(nodes))(*[_NodeModel(*map(float, nd)) for nd in nodes])
    return arr, _CommModel(*map(float, comm))


def node_time(node, comm, b: float) -> float:
    nd = _NodeModel(*map(float, node))
    cm = _CommModel(*map(float, comm))
    return lib().cannikin_node_time(ctypes.byref(nd), ctypes.byref(cm), float(b))


def opt_split(nodes, comm, B: int, lo=None, cap=None, round_paper: bool = False) -> dict:
    n = len(nodes)
    arr, cm = _models(nodes, comm)
    b = (ctypes.c_int64 * n)()
    br = (ctypes.c_double * n)()
    t = (ctypes.c_double * 2)()
    lab = (ctypes.c_int * n)()
    _check(lib().cannikin_opt_split(arr, n, ctypes.byref(cm), int(B),
                                    _i64(lo) if lo is not None else None,
                                    _i64(cap) if cap is not None else None,
                                    ROUND_PAPER if round_paper else 0, b, br, t, lab))
    return {"b": list(b), "b_real": list(br), "T_real": t[0], "T_int": t[1], "labels": list(lab)}


def warmup_split(t_sample, B: int):
    n = len(t_sample)
    br = (ctypes.c_double * n)()
    b = (ctypes.c_int64 * n)()
    _check(lib().cannikin_warmup_split(_dbl(t_sample), n, int(B), br, b))
    return list(b), list(br)


# ----------------------------------------------------------------------------- measured-model loop
def fit_linear(x, y):
    sl, ic = ctypes.c_double(), ctypes.c_double()
    _check(lib().cannikin_fit_linear(_dbl(x), _dbl(y), len(x), ctypes.byref(sl), ctypes.byref(ic)))
    return sl.value, ic.value


def ivw(estimates, variances) -> float:
    out = ctypes.c_double()
    _check(lib().cannikin_ivw(_dbl(estimates), _dbl(variances), len(estimates), ctypes.byref(out)))
    return out.value


class Analyzer:
    """The paper's analyzer/optimizer loop: observe timings, plan each epoch."""

    def __init__(self, n: int):
        h = ctypes.c_void_p()
        _check(lib().cannikin_analyzer_create(n, ctypes.byref(h)))
        self._h, self.n = h, n

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                lib().cannikin_analyzer_destroy(self._h)
                self._h = None
        except Exception:
            pass

    def observe(self, node: int, it: int, b: int, a: float, P: float, gamma: float, t_o: float,
                t_u: float):
        _check(lib().cannikin_analyzer_observe(self._h, node, int(it), int(b), float(a), float(P),
                                               float(gamma), float(t_o), float(t_u)))

    def models(self):
        nodes = (_NodeModel * self.n)()
        cm = _CommModel()
        _check(lib().cannikin_analyzer_models(self._h, nodes, ctypes.byref(cm)))
        return [(x.q, x.s, x.k, x.m) for x in nodes], (cm.gamma, cm.t_o, cm.t_u)

    def choose_batch(self, candidates, B0: int, B_noise: float):
        """Goodput-optimal total batch with the OptPerf_init cache."""
        Bo = ctypes.c_int64()
        b = (ctypes.c_int64 * self.n)()
        t = ctypes.c_double()
        full = ctypes.c_int()
        _check(lib().cannikin_analyzer_choose_batch(self._h, _i64(candidates), len(candidates),
                                                    int(B0), float(B_noise), ctypes.byref(Bo), b,
                                                    ctypes.byref(t), ctypes.byref(full)))
        return {"B": Bo.value, "b": list(b), "T_pred": t.value, "full_recompute": bool(full.value)}

    def plan(self, B: int, cap=None):
        b = (ctypes.c_int64 * self.n)()
        t = ctypes.c_double()
        ph = ctypes.c_int()
        _check(lib().cannikin_analyzer_plan(self._h, int(B), _i64(cap) if cap is not None else None,
                                            b, ctypes.byref(t), ctypes.byref(ph)))
        return {"b": list(b), "T_pred": t.value, "phase": ph.value}


# ----------------------------------------------------------------------------- adaptive batch
class GnsEma:
    """EMA of the aggregated G and S (separately), B_noise = S / G of the averages."""

    def __init__(self, decay: float = 0.9):
        self._s = _GnsEma(0.0, 0.0, float(decay), 0, float("nan"))

    def update(self, G2: float, trS: float):
        _check(lib().cannikin_gns_ema_update(ctypes.byref(self._s), float(G2), float(trS)))

    @property
    def count(self) -> int:
        return self._s.count

    @property
    def B_noise(self) -> float:
        """S / G of the averages, as cannikin_gns_ema_update last set it (NaN before any)."""
        return self._s.B_noise


def efficiency(B: int, B0: int, B_noise: float) -> float:
    return lib().cannikin_efficiency(int(B), int(B0), float(B_noise))


def choose_batch(nodes, comm, candidates, B0: int, B_noise: float):
    arr, cm = _models(nodes, comm)
    k = len(candidates)
    Bo = ctypes.c_int64()
    T = (ctypes.c_double * k)()
    G = (ctypes.c_double * k)()
    _check(lib().cannikin_choose_batch(arr, len(nodes), ctypes.byref(cm), _i64(candidates), k,
                                       int(B0), float(B_noise), ctypes.byref(Bo), T, G))
    return {"B": Bo.value, "T": list(T), "goodput": list(G)}


class ControlStep:
    """The host half of a training step in one native call: GNS estimate + EMA + next split.
    Buffers are prepared once; call(stats_ptr) with the address of n+1 float64 statistics
    (e.g. a pinned host tensor's data_ptr())."""

    def __init__(self, b, nodes, comm, B_next: int, decay: float = 0.9):
        self.n = len(b)
        self._b = _i64(b)
        self._nodes, self._cm = _models(nodes, comm)
        self._ema = _GnsEma(0.0, 0.0, float(decay), 0, float("nan"))
        self._res = _GnsResult()
        self._bn = (ctypes.c_int64 * self.n)()
        self._t = ctypes.c_double()
        self.B_next = int(B_next)
        self._f = lib().cannikin_control_step

    def __call__(self, stats_ptr: int):
        st = self._f(ctypes.cast(stats_ptr, _DP), self._b, self.n, ctypes.byref(self._ema),
                     self._nodes, ctypes.byref(self._cm), self.B_next, ctypes.byref(self._res),
                     self._bn, ctypes.byref(self._t))
        if st:
            _check(st)
        return self._res.B_noise

    @property
    def result(self):
        n = self.n
        r = self._res
        return {"G2": r.G2, "trS": r.trS, "B_noise": r.B_noise, "wG": list(r.wG[:n]),
                "wS": list(r.wS[:n]), "b_next": list(self._bn), "T_next": self._t.value,
                "ema_B_noise": self._ema.B_noise}
