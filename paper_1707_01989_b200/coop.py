"""Thin ctypes binding of libcoop (include/coop.h) -- argument marshalling only.

Every step of the BFS/SSSP path runs inside the library's CUDA kernels; this
module only converts torch tensors to device pointers and fills the C
structs.  There is no CPU fallback: if libcoop.so is missing or the device is
not a CUDA GPU, calls raise.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libcoop.so")

# ---- enums (coop.h)
COOP_OK = 0
STATUS_NAMES = {0: "COOP_OK", 1: "COOP_ERR_INVALID_ARG", 2: "COOP_ERR_CUDA", 3: "COOP_ERR_NOT_CORESIDENT",
                4: "COOP_ERR_FORK_BOUND", 5: "COOP_ERR_NO_CAPACITY", 6: "COOP_ERR_TIMEOUT",
                7: "COOP_ERR_OVERFLOW", 8: "COOP_ERR_NCCL", 9: "COOP_ERR_INVARIANT", 10: "COOP_ERR_BUSY"}
BARRIER_QUERY, BARRIER_PLAIN, BARRIER_NAIVE = 0, 1, 2
POLICY_NEVER, POLICY_SCRIPTED, POLICY_RANDOM, POLICY_SCHEDULER = 0, 1, 2, 3
FLAG_CHECK = 0x1
FLAG_DIROPT = 0x2


class CoopError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class CooperativeCSR(ctypes.Structure):
    _fields_ = [("num_vertices", ctypes.c_int64), ("num_edges", ctypes.c_int64),
                ("row_offsets", ctypes.c_void_p), ("offset_bits", ctypes.c_int32),
                ("col_idx", ctypes.c_void_p), ("weights", ctypes.c_void_p),
                ("max_weight", ctypes.c_uint32), ("probe", ctypes.c_void_p), ("isolated", ctypes.c_void_p)]


class Opts(ctypes.Structure):
    _fields_ = [("max_wgs", ctypes.c_uint32), ("init_wgs", ctypes.c_uint32),
                ("threads_per_wg", ctypes.c_uint32), ("barrier_mode", ctypes.c_uint32),
                ("barriers_per_level", ctypes.c_uint32), ("policy", ctypes.c_uint32),
                ("script", ctypes.POINTER(ctypes.c_uint32)), ("script_len", ctypes.c_uint32),
                ("flags", ctypes.c_uint32), ("seed", ctypes.c_uint64), ("resize_prob", ctypes.c_double),
                ("task_wgs", ctypes.c_uint32), ("task_blocks", ctypes.c_uint32),
                ("task_block_ns", ctypes.c_uint64), ("task_period_ns", ctypes.c_uint64),
                ("task_first_ns", ctypes.c_uint64), ("task_max", ctypes.c_uint32),
                ("timeout_ns", ctypes.c_uint64), ("stream", ctypes.c_void_p),
                ("ev_kernel_start", ctypes.c_void_p), ("ev_kernel_end", ctypes.c_void_p),
                ("workspace", ctypes.c_uint32), ("sssp_delta", ctypes.c_uint32),
                ("bfs_alpha", ctypes.c_uint32), ("bfs_beta", ctypes.c_uint32)]


class TaskEvent(ctypes.Structure):
    _fields_ = [("t_arrive", ctypes.c_uint64), ("t_first_surrender", ctypes.c_uint64),
                ("t_last_surrender", ctypes.c_uint64), ("t_first_start", ctypes.c_uint64),
                ("t_end", ctypes.c_uint64), ("demanded", ctypes.c_uint32), ("surrendered", ctypes.c_uint32)]


class Stats(ctypes.Structure):
    _fields_ = [("kernel_ns", ctypes.c_uint64), ("edges_scanned", ctypes.c_uint64),
                ("frontier_total", ctypes.c_uint64), ("reached", ctypes.c_uint64),
                ("levels", ctypes.c_uint32), ("episodes", ctypes.c_uint32),
                ("kills", ctypes.c_uint32), ("forks", ctypes.c_uint32),
                ("min_m", ctypes.c_uint32), ("max_m", ctypes.c_uint32),
                ("n_wgs", ctypes.c_uint32), ("threads_per_wg", ctypes.c_uint32),
                ("tasks_posted", ctypes.c_uint32), ("tasks_completed", ctypes.c_uint32),
                ("bottom_up_levels", ctypes.c_uint32), ("mid_kills", ctypes.c_uint32),
                ("handbacks", ctypes.c_uint32), ("replays", ctypes.c_uint32), ("reserved0", ctypes.c_uint32),
                ("m_trace", ctypes.POINTER(ctypes.c_uint32)), ("m_trace_cap", ctypes.c_uint32),
                ("level_sizes", ctypes.POINTER(ctypes.c_uint32)), ("level_sizes_cap", ctypes.c_uint32),
                ("level_end_ns", ctypes.POINTER(ctypes.c_uint64)), ("level_end_ns_cap", ctypes.c_uint32),
                ("task_events", ctypes.POINTER(TaskEvent)), ("task_events_cap", ctypes.c_uint32)]


class DeviceInfo(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int), ("sm_count", ctypes.c_int), ("max_ctas_per_sm", ctypes.c_int),
                ("max_coresident", ctypes.c_int), ("regs_per_thread", ctypes.c_int),
                ("l2_bytes", ctypes.c_size_t), ("hbm_bytes", ctypes.c_size_t)]


class BarrierStats(ctypes.Structure):
    _fields_ = [("iters", ctypes.c_uint64), ("ns_per_barrier", ctypes.c_double), ("kernel_ns", ctypes.c_uint64),
                ("kills", ctypes.c_uint32), ("forks", ctypes.c_uint32), ("violations", ctypes.c_uint32)]


class CoopPart(ctypes.Structure):
    """coop_part (1-D partitioned BFS, one rank)."""
    _fields_ = [("num_vertices", ctypes.c_int64), ("v_begin", ctypes.c_int64), ("v_end", ctypes.c_int64),
                ("rank", ctypes.c_int32), ("nranks", ctypes.c_int32), ("seq", ctypes.c_uint32),
                ("row_offsets", ctypes.c_void_p), ("offset_bits", ctypes.c_int32),
                ("col_local", ctypes.c_void_p), ("num_edges", ctypes.c_int64),
                ("hub_ids", ctypes.c_void_p), ("hub_prefix", ctypes.c_void_p),
                ("num_hubs", ctypes.c_uint32), ("hub_degree", ctypes.c_uint32),
                ("frontier", (ctypes.c_void_p * 2) * 8), ("flags", ctypes.c_void_p * 8),
                ("rows_offsets", ctypes.c_void_p), ("rows_col", ctypes.c_void_p),
                ("num_edges_global", ctypes.c_int64)]


class DevOpts(ctypes.Structure):
    _fields_ = [("max_wgs", ctypes.c_uint32), ("init_wgs", ctypes.c_uint32), ("policy", ctypes.c_uint32),
                ("flags", ctypes.c_uint32), ("seed", ctypes.c_uint64), ("resize_prob", ctypes.c_double),
                ("kill_prob", ctypes.c_double), ("fork_prob", ctypes.c_double), ("max_fork", ctypes.c_uint32),
                ("script", ctypes.POINTER(ctypes.c_uint32)), ("script_len", ctypes.c_uint32),
                ("m_trace_cap", ctypes.c_uint32), ("timeout_ns", ctypes.c_uint64)]


class DevStats(ctypes.Structure):
    _fields_ = [("kernel_ns", ctypes.c_uint64), ("n_wgs", ctypes.c_uint32), ("kills", ctypes.c_uint32),
                ("forks", ctypes.c_uint32), ("episodes", ctypes.c_uint32), ("barriers", ctypes.c_uint32),
                ("offers", ctypes.c_uint32), ("fork_calls", ctypes.c_uint32), ("min_m", ctypes.c_uint32),
                ("max_m", ctypes.c_uint32), ("final_m", ctypes.c_uint32), ("violations", ctypes.c_uint32),
                ("m_trace", ctypes.POINTER(ctypes.c_uint32)), ("m_trace_cap", ctypes.c_uint32)]


class WsTree(ctypes.Structure):
    _fields_ = [("seed", ctypes.c_uint64), ("depth", ctypes.c_uint32), ("max_fanout", ctypes.c_uint32),
                ("fixed", ctypes.c_uint32), ("rounds", ctypes.c_uint32), ("queue_cap", ctypes.c_uint32)]


class WsResult(ctypes.Structure):
    _fields_ = [("count", ctypes.c_uint64), ("total", ctypes.c_uint64), ("hist", ctypes.c_uint64 * 64),
                ("steals", ctypes.c_uint64)]


# every function declared in include/coop.h: name -> (restype, argtypes)
_P = ctypes.c_void_p
# bottom-up BFS probe records (coop_csr.probe), built once per graph; COOP_PROBE=0 disables (A/B)
USE_PROBE = os.environ.get("COOP_PROBE", "1") != "0"
# BFS graphs get a hub-first copy of their neighbour lists (coop_csr_hub_first); COOP_HUB_FIRST=0 disables
USE_HUB_FIRST = os.environ.get("COOP_HUB_FIRST", "1") != "0"
SIGNATURES = {
    "coop_abi_version": (ctypes.c_int, []),
    "coop_status_string": (ctypes.c_char_p, [ctypes.c_int]),
    "coop_last_error": (ctypes.c_char_p, []),
    "coop_device_query": (ctypes.c_int, [ctypes.c_int, ctypes.c_uint32, ctypes.POINTER(DeviceInfo)]),
    "coop_csr_probe": (ctypes.c_int, [ctypes.POINTER(CooperativeCSR), _P, _P]),
    "coop_csr_hub_first": (ctypes.c_int, [ctypes.POINTER(CooperativeCSR), _P, _P]),
    "coop_csr_isolated": (ctypes.c_int, [ctypes.POINTER(CooperativeCSR), _P, _P]),
    "coop_bfs": (ctypes.c_int, [ctypes.POINTER(CooperativeCSR), ctypes.c_int64, _P, ctypes.POINTER(Opts),
                                ctypes.POINTER(Stats)]),
    "coop_sssp": (ctypes.c_int, [ctypes.POINTER(CooperativeCSR), ctypes.c_int64, _P, ctypes.POINTER(Opts),
                                 ctypes.POINTER(Stats)]),
    "coop_bfs_host": (ctypes.c_int, [ctypes.c_int64, _P, ctypes.c_int32, _P, ctypes.c_int64, _P,
                                     ctypes.POINTER(Opts), ctypes.POINTER(Stats)]),
    "coop_sssp_host": (ctypes.c_int, [ctypes.c_int64, _P, ctypes.c_int32, _P, _P, ctypes.c_uint32,
                                      ctypes.c_int64, _P, ctypes.POINTER(Opts), ctypes.POINTER(Stats)]),
    "coop_barrier_bench": (ctypes.c_int, [ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_double,
                                          ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32,
                                          ctypes.POINTER(BarrierStats)]),
    "coop_l2_atomic_rtt": (ctypes.c_int, [ctypes.c_uint64, ctypes.POINTER(ctypes.c_double)]),
    "coop_l2_latency_profile": (ctypes.c_int, [ctypes.c_uint64, ctypes.POINTER(ctypes.c_double)]),
    "coop_debug_trace": (ctypes.c_int, [ctypes.POINTER(ctypes.c_uint64)]),
    "coop_launch": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(CooperativeCSR), ctypes.c_int64, _P,
                                   ctypes.POINTER(Opts), ctypes.POINTER(_P)]),
    "coop_submit_task": (ctypes.c_int, [_P, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint64,
                                        ctypes.POINTER(ctypes.c_uint64)]),
    "coop_demand": (ctypes.c_int, [_P, ctypes.c_uint32]),
    "coop_grant": (ctypes.c_int, [_P, ctypes.c_uint32]),
    "coop_query": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_uint32)]),
    "coop_current_m": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_uint32)]),
    "coop_wait": (ctypes.c_int, [_P, ctypes.POINTER(Stats)]),
    "coop_destroy": (None, [_P]),
    "coop_bfs_part": (ctypes.c_int, [ctypes.POINTER(CoopPart), ctypes.c_int64, _P, ctypes.POINTER(Opts),
                                     ctypes.POINTER(Stats)]),
    "coop_bfs_part_launch": (ctypes.c_int, [ctypes.POINTER(CoopPart), ctypes.c_int64, _P, ctypes.POINTER(Opts),
                                            ctypes.POINTER(_P)]),
    "coop_spin_task": (ctypes.c_int, [ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint64, _P]),
    "coop_bfs_launch": (ctypes.c_int, [ctypes.POINTER(CooperativeCSR), ctypes.c_int64, _P, ctypes.POINTER(Opts),
                                       ctypes.POINTER(_P)]),
    "coop_bfs_loop": (ctypes.c_int, [ctypes.POINTER(CooperativeCSR), _P, ctypes.c_uint32, ctypes.c_uint64, _P,
                                     ctypes.POINTER(ctypes.c_uint64), ctypes.c_uint32,
                                     ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(Opts), ctypes.POINTER(Stats)]),
    "coop_sssp_part": (ctypes.c_int, [ctypes.POINTER(CoopPart), _P, ctypes.c_int64, _P, ctypes.POINTER(Opts),
                                      ctypes.POINTER(Stats)]),
    "coop_sssp_part_launch": (ctypes.c_int, [ctypes.POINTER(CoopPart), _P, ctypes.c_int64, _P, ctypes.POINTER(Opts),
                                             ctypes.POINTER(_P)]),
    "coop_bfs_part_nccl": (ctypes.c_int, [ctypes.POINTER(CoopPart), ctypes.c_int64, _P, _P, ctypes.POINTER(Opts),
                                          ctypes.POINTER(Stats)]),
    "coop_nccl_get_unique_id": (ctypes.c_int, [_P]),
    "coop_nccl_comm_init": (ctypes.c_int, [ctypes.c_int32, _P, ctypes.c_int32, ctypes.POINTER(_P)]),
    "coop_nccl_comm_destroy": (ctypes.c_int, [_P]),
    "coop_exchange_alloc": (ctypes.c_int, [ctypes.c_uint64, ctypes.POINTER(_P)]),
    "coop_exchange_free": (ctypes.c_int, [_P]),
    "coop_ipc_get_handle": (ctypes.c_int, [_P, _P]),
    "coop_ipc_open": (ctypes.c_int, [_P, ctypes.POINTER(_P)]),
    "coop_ipc_close": (ctypes.c_int, [_P]),
    "coop_dev_create": (ctypes.c_int, [ctypes.POINTER(DevOpts), ctypes.POINTER(_P)]),
    "coop_dev_arm": (ctypes.c_int, [_P, ctypes.c_uint32, _P, ctypes.POINTER(_P)]),
    "coop_dev_demand": (ctypes.c_int, [_P, ctypes.c_uint32]),
    "coop_dev_grant": (ctypes.c_int, [_P, ctypes.c_uint32]),
    "coop_dev_collect": (ctypes.c_int, [_P, _P, ctypes.POINTER(DevStats)]),
    "coop_dev_destroy": (None, [_P]),
    "coop_color": (ctypes.c_int, [_P, ctypes.POINTER(CooperativeCSR), ctypes.c_uint64, _P, ctypes.c_uint32,
                                  ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(DevStats)]),
    "coop_mis": (ctypes.c_int, [_P, ctypes.POINTER(CooperativeCSR), ctypes.c_uint64, _P, ctypes.c_uint32,
                                ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(DevStats)]),
    "coop_psssp": (ctypes.c_int, [_P, ctypes.POINTER(CooperativeCSR), ctypes.c_int64, _P, ctypes.c_uint32,
                                  ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(DevStats)]),
    "coop_fig4_bfs": (ctypes.c_int, [_P, ctypes.POINTER(CooperativeCSR), ctypes.c_int64, _P, ctypes.c_uint32,
                                     ctypes.POINTER(DevStats)]),
    "coop_work_steal": (ctypes.c_int, [_P, ctypes.POINTER(WsTree), ctypes.c_uint32, ctypes.POINTER(WsResult),
                                       ctypes.POINTER(DevStats)]),
}

_lib = None


def load(path: str = LIB_PATH):
    """Load libcoop.so (raises if it has not been built -- no fallback)."""
    global _lib
    if _lib is None:
        if path == LIB_PATH and os.environ.get("COOP_LIB"):   # a build variant (tools/, experiments)
            path = os.path.abspath(os.environ["COOP_LIB"])
        if not os.path.exists(path):
            raise RuntimeError(f"{path} not built: run `python -m paper_1707_01989_b200.build` "
                               "(or __graft_entry__.build()); there is no CPU fallback")
        lib = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            if path != LIB_PATH and not hasattr(lib, name):
                continue        # an older build variant (tools/): only what it exports is usable
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def _check(rc: int):
    if rc != COOP_OK:
        raise CoopError(rc, load().coop_last_error().decode(errors="replace"))


# ---------------------------------------------------------------- helpers
@dataclass
class RunStats:
    kernel_ns: int = 0
    edges_scanned: int = 0
    frontier_total: int = 0
    reached: int = 0
    levels: int = 0
    episodes: int = 0
    kills: int = 0
    forks: int = 0
    min_m: int = 0
    max_m: int = 0
    n_wgs: int = 0
    threads_per_wg: int = 0
    tasks_posted: int = 0
    tasks_completed: int = 0
    bottom_up_levels: int = 0
    mid_kills: int = 0
    handbacks: int = 0
    replays: int = 0
    m_trace: list = field(default_factory=list)
    level_sizes: list = field(default_factory=list)
    level_end_ns: list = field(default_factory=list)
    task_events: list = field(default_factory=list)


def with_offset_bits(g, bits: int):
    """A view of graphgen.CSR ``g`` whose row offsets go to the library as ``bits``-bit
    integers (64 is chosen automatically only when E >= 2^32, e.g. RMAT-27 on one GPU;
    forcing it on small graphs exercises that path)."""
    if bits not in (32, 64):
        raise ValueError("offset_bits must be 32 or 64")
    h = type(g)(g.num_vertices, g.row_offsets, g.col_idx, g.weights, g.name)
    if getattr(g, "max_weight", None) is not None:
        h.max_weight = g.max_weight
    h.offset_bits = bits
    return h


def _bfs_csr(g):
    """The BFS layout of a graph: hub-first neighbour lists (coop_csr_hub_first) and the probe
    records built from them -- graph-layout steps done once per graph and cached on it."""
    import torch
    cache = getattr(g, "_coop_bfs_cache", None)
    if cache is not None:
        return cache
    c0, keep0 = _device_csr(g, need_weights=False, probe=not USE_HUB_FIRST)
    if not USE_HUB_FIRST or g.num_edges == 0 or g.num_edges >= (1 << 31) - 1:
        res = (c0, keep0)
    else:
        col2 = torch.empty_like(keep0[1])
        _check(load().coop_csr_hub_first(ctypes.byref(c0), col2.data_ptr(), None))
        c = CooperativeCSR(c0.num_vertices, c0.num_edges, c0.row_offsets, c0.offset_bits, col2.data_ptr(), None,
                           0, None, None)
        probe = None
        if USE_PROBE:
            probe = torch.empty(g.num_vertices, dtype=torch.int64, device=col2.device)
            _check(load().coop_csr_probe(ctypes.byref(c), probe.data_ptr(), None))
            c.probe = probe.data_ptr()
        iso = torch.empty((g.num_vertices + 31) // 32, dtype=torch.int32, device=col2.device)
        _check(load().coop_csr_isolated(ctypes.byref(c), iso.data_ptr(), None))
        c.isolated = iso.data_ptr()
        res = (c, (keep0[0], col2, None, probe, iso))
    try:
        g._coop_bfs_cache = res
    except AttributeError:
        pass
    return res


def _device_csr(g, need_weights: bool, probe: bool = True):
    """graphgen.CSR on a CUDA device -> (CooperativeCSR, keepalive tensors)."""
    import torch
    if not g.col_idx.is_cuda:
        raise ValueError("graph tensors must be on a CUDA device (use coop_bfs_host for host arrays)")
    cache = getattr(g, "_coop_cache", None)
    if cache is not None and (cache[2] is not None or not need_weights):
        return cache[0], cache[1]
    E = g.num_edges
    if E < (1 << 32) and getattr(g, "offset_bits", None) != 64:
        ro = g.row_offsets.to(torch.int32) if g.row_offsets.dtype != torch.int32 else g.row_offsets
        bits = 32
    else:
        ro = g.row_offsets.to(torch.int64)
        bits = 64
    ro = ro.contiguous()
    col = g.col_idx.to(torch.int32).contiguous()
    w = None
    if need_weights:
        if g.weights is None:
            raise ValueError("SSSP needs weights")
        w = g.weights.to(torch.int32).contiguous()
    c = CooperativeCSR(g.num_vertices, E, ro.data_ptr(), bits, col.data_ptr() if E else None,
                       w.data_ptr() if (w is not None and E) else None,
                       int(getattr(g, "max_weight", 0) or 0), None, None)
    probe_t = None
    if probe and USE_PROBE and g.num_vertices > 0:
        # graph layout step (once per graph, like the CSR conversion above): per-vertex
        # {degree | first neighbour} records for the bottom-up BFS levels
        probe_t = torch.empty(g.num_vertices, dtype=torch.int64, device=col.device)
        _check(load().coop_csr_probe(ctypes.byref(c), probe_t.data_ptr(), None))
        c.probe = probe_t.data_ptr()
    keep = (ro, col, w, probe_t)
    try:
        g._coop_cache = (c, keep, w)   # converted arrays are reused by later calls
    except AttributeError:
        pass
    return c, keep


def make_opts(*, max_wgs=0, init_wgs=0, threads_per_wg=0, barrier_mode=BARRIER_QUERY, barriers_per_level=1,
              policy=POLICY_NEVER, script: Optional[Sequence[int]] = None, flags=0, seed=0, resize_prob=0.0,
              task_wgs=0, task_blocks=0, task_block_ns=0, task_period_ns=0, task_first_ns=0, task_max=0,
              timeout_ns=0, stream=None, ev_kernel_start=None, ev_kernel_end=None, workspace=0, sssp_delta=0,
              bfs_alpha=0, bfs_beta=0):
    import torch
    o = Opts()
    o.max_wgs, o.init_wgs, o.threads_per_wg = max_wgs, init_wgs, threads_per_wg
    o.barrier_mode, o.barriers_per_level, o.policy = barrier_mode, barriers_per_level, policy
    keep = None
    if script is not None:
        keep = (ctypes.c_uint32 * len(script))(*script)
        o.script = ctypes.cast(keep, ctypes.POINTER(ctypes.c_uint32))
        o.script_len = len(script)
    o.flags, o.seed, o.resize_prob = flags, seed, resize_prob
    o.task_wgs, o.task_blocks, o.task_block_ns = task_wgs, task_blocks, task_block_ns
    o.task_period_ns, o.task_first_ns, o.task_max = task_period_ns, task_first_ns, task_max
    o.timeout_ns = timeout_ns
    if stream is None and torch.cuda.is_available():
        stream = torch.cuda.current_stream().cuda_stream
    o.stream = stream
    o.workspace = workspace
    o.sssp_delta = sssp_delta
    o.bfs_alpha, o.bfs_beta = bfs_alpha, bfs_beta
    if ev_kernel_start is not None:   # torch.cuda.Event(enable_timing=True)
        o.ev_kernel_start = ev_kernel_start.cuda_event
        o.ev_kernel_end = ev_kernel_end.cuda_event
    return o, keep


def _stats_struct(trace_cap=0, level_cap=0, event_cap=0):
    st = Stats()
    bufs = {}
    if trace_cap:
        bufs["m"] = (ctypes.c_uint32 * trace_cap)()
        st.m_trace, st.m_trace_cap = ctypes.cast(bufs["m"], ctypes.POINTER(ctypes.c_uint32)), trace_cap
    if level_cap:
        bufs["l"] = (ctypes.c_uint32 * level_cap)()
        st.level_sizes, st.level_sizes_cap = ctypes.cast(bufs["l"], ctypes.POINTER(ctypes.c_uint32)), level_cap
        bufs["t"] = (ctypes.c_uint64 * level_cap)()
        st.level_end_ns, st.level_end_ns_cap = ctypes.cast(bufs["t"], ctypes.POINTER(ctypes.c_uint64)), level_cap
    if event_cap:
        bufs["e"] = (TaskEvent * event_cap)()
        st.task_events, st.task_events_cap = ctypes.cast(bufs["e"], ctypes.POINTER(TaskEvent)), event_cap
    return st, bufs


def _to_runstats(st: Stats, bufs) -> RunStats:
    r = RunStats(**{k: getattr(st, k) for k in ("kernel_ns", "edges_scanned", "frontier_total", "reached",
                                                "levels", "episodes", "kills", "forks", "min_m", "max_m",
                                                "n_wgs", "threads_per_wg", "tasks_posted", "tasks_completed",
                                                "bottom_up_levels", "mid_kills", "handbacks", "replays")})
    if "m" in bufs:
        r.m_trace = list(bufs["m"][: min(st.episodes, st.m_trace_cap)])
    if "l" in bufs:
        r.level_sizes = list(bufs["l"][: min(st.levels, st.level_sizes_cap)])
        r.level_end_ns = list(bufs["t"][: min(st.levels, st.level_end_ns_cap)])
    if "e" in bufs:
        n = min(st.tasks_posted, st.task_events_cap)
        r.task_events = [{f: getattr(bufs["e"][i], f) for f, _ in TaskEvent._fields_} for i in range(n)]
    return r


# ---------------------------------------------------------------- public API
def bfs(g, source: int, levels_out=None, *, trace_cap=0, level_cap=0, event_cap=0, **opts):
    """Cooperative BFS on the current CUDA device.  Returns (levels int32 tensor, RunStats)."""
    import torch
    lib = load()
    c, keep = _bfs_csr(g)
    if levels_out is None:
        levels_out = torch.empty(g.num_vertices, dtype=torch.int32, device=g.col_idx.device)
    o, k2 = make_opts(**opts)
    st, bufs = _stats_struct(trace_cap, level_cap, event_cap)
    _check(lib.coop_bfs(ctypes.byref(c), int(source), levels_out.data_ptr(), ctypes.byref(o), ctypes.byref(st)))
    del keep, k2
    return levels_out, _to_runstats(st, bufs)


class BfsCall:
    """An asynchronous cooperative BFS (coop_bfs_launch); wait() returns RunStats."""

    def __init__(self, g, source: int, levels_out, **opts):
        lib = load()
        self._c, self._keep = _bfs_csr(g)
        self._o, self._k2 = make_opts(**opts)
        self.h = ctypes.c_void_p()
        self.out = levels_out
        _check(lib.coop_bfs_launch(ctypes.byref(self._c), int(source), levels_out.data_ptr(), ctypes.byref(self._o),
                                   ctypes.byref(self.h)))

    def wait(self, *, level_cap=0) -> "RunStats":
        lib = load()
        st, bufs = _stats_struct(0, level_cap, 0)
        rc = lib.coop_wait(self.h, ctypes.byref(st))
        lib.coop_destroy(self.h)
        self.h = None
        _check(rc)
        return _to_runstats(st, bufs)


def bfs_loop(g, sources, loop_s: float, levels_out=None, *, run_cap=1 << 20, event_cap=0, **opts):
    """BFS looped over ``sources`` inside one persistent launch for ``loop_s`` seconds
    (coop_bfs_loop).  Returns (levels of the last run, runs, run end times in s after
    the kernel start, RunStats)."""
    import numpy as np
    import torch
    lib = load()
    c, keep = _bfs_csr(g)
    dev = g.col_idx.device
    src = torch.as_tensor(list(sources), dtype=torch.int64, device=dev)
    if levels_out is None:
        levels_out = torch.empty(g.num_vertices, dtype=torch.int32, device=dev)
    o, k2 = make_opts(**opts)
    st, bufs = _stats_struct(0, 0, event_cap)
    t = np.zeros(run_cap, dtype=np.uint64)
    runs = ctypes.c_uint32()
    _check(lib.coop_bfs_loop(ctypes.byref(c), src.data_ptr(), src.numel(), int(loop_s * 1e9), levels_out.data_ptr(),
                             t.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), run_cap, ctypes.byref(runs),
                             ctypes.byref(o), ctypes.byref(st)))
    del keep, k2
    n = runs.value
    return levels_out, n, t[: min(n, run_cap)].astype(np.float64) * 1e-9, _to_runstats(st, bufs)


def sssp(g, source: int, dist_out=None, *, trace_cap=0, level_cap=0, event_cap=0, **opts):
    """Cooperative worklist SSSP.  Returns (dist int32 tensor holding uint32 bits, RunStats)."""
    import torch
    lib = load()
    c, keep = _device_csr(g, need_weights=True)
    if dist_out is None:
        dist_out = torch.empty(g.num_vertices, dtype=torch.int32, device=g.col_idx.device)
    o, k2 = make_opts(**opts)
    st, bufs = _stats_struct(trace_cap, level_cap, event_cap)
    _check(lib.coop_sssp(ctypes.byref(c), int(source), dist_out.data_ptr(), ctypes.byref(o), ctypes.byref(st)))
    del keep, k2
    return dist_out, _to_runstats(st, bufs)


def bfs_host(ro, col, source: int, levels_out, **opts):
    """End-to-end BFS from HOST arrays (pinned torch CPU tensors or numpy): H2D, kernel, D2H in the call."""
    lib = load()
    V = ro.numel() - 1
    bits = 32 if ro.element_size() == 4 else 64
    o, k2 = make_opts(**opts)
    st, bufs = _stats_struct()
    _check(lib.coop_bfs_host(V, ro.data_ptr(), bits, col.data_ptr(), int(source), levels_out.data_ptr(),
                             ctypes.byref(o), ctypes.byref(st)))
    return levels_out, _to_runstats(st, bufs)


def sssp_host(ro, col, w, max_weight: int, source: int, dist_out, **opts):
    lib = load()
    V = ro.numel() - 1
    bits = 32 if ro.element_size() == 4 else 64
    o, k2 = make_opts(**opts)
    st, bufs = _stats_struct()
    _check(lib.coop_sssp_host(V, ro.data_ptr(), bits, col.data_ptr(), w.data_ptr(), int(max_weight),
                              int(source), dist_out.data_ptr(), ctypes.byref(o), ctypes.byref(st)))
    return dist_out, _to_runstats(st, bufs)


def barrier_bench(n_ctas: int, iters: int, *, threads=128, resize_prob=0.0, seed=3, plain=False, check=False):
    lib = load()
    out = BarrierStats()
    _check(lib.coop_barrier_bench(n_ctas, threads, iters, resize_prob, seed,
                                  BARRIER_PLAIN if plain else BARRIER_QUERY, FLAG_CHECK if check else 0,
                                  ctypes.byref(out)))
    return {f: getattr(out, f) for f, _ in BarrierStats._fields_}


def l2_latency_profile(iters: int = 20000) -> dict:
    """ns per dependent operation, per kind, on 8 SMs (coop_l2_latency_profile)."""
    lib = load()
    buf = (ctypes.c_double * 32)()
    _check(lib.coop_l2_latency_profile(iters, buf))
    names = ["atom_relaxed_u64", "atom_relaxed_u32", "atom_acq_rel_u64", "ld_acquire_u64"]
    out = {}
    for k, n in enumerate(names):
        v = sorted(x for x in buf[8 * k: 8 * k + 8] if x > 0)
        out[n] = {"min": v[0], "median": v[len(v) // 2], "max": v[-1], "sms": len(v)} if v else None
    return out


def l2_atomic_rtt(iters: int = 100000) -> float:
    lib = load()
    v = ctypes.c_double()
    _check(lib.coop_l2_atomic_rtt(iters, ctypes.byref(v)))
    return v.value


def debug_trace() -> list:
    """Barrier phase breakdown of the last call (COOP_TRACE builds only)."""
    buf = (ctypes.c_uint64 * 16)()
    _check(load().coop_debug_trace(buf))
    return list(buf)


def device_query(device: int = 0, threads_per_wg: int = 512) -> dict:
    lib = load()
    d = DeviceInfo()
    _check(lib.coop_device_query(device, threads_per_wg, ctypes.byref(d)))
    return {f: getattr(d, f) for f, _ in DeviceInfo._fields_}


class Handle:
    """Asynchronous cooperative kernel (coop_launch) with the host->GPU channel."""

    def __init__(self, kind: str, g, source: int, out, **opts):
        lib = load()
        self._c, self._keep = _device_csr(g, need_weights=(kind == "sssp"))
        self._o, self._k2 = make_opts(policy=POLICY_SCHEDULER, **opts)
        self.out = out
        h = ctypes.c_void_p()
        _check(lib.coop_launch(0 if kind == "bfs" else 1, ctypes.byref(self._c), int(source), out.data_ptr(),
                               ctypes.byref(self._o), ctypes.byref(h)))
        self._h = h

    def submit_task(self, wgs: int, blocks: int, block_ns: int) -> int:
        tid = ctypes.c_uint64()
        _check(load().coop_submit_task(self._h, wgs, blocks, block_ns, ctypes.byref(tid)))
        return tid.value

    def demand(self, n: int):
        _check(load().coop_demand(self._h, n))

    def grant(self, n: int):
        _check(load().coop_grant(self._h, n))

    def query(self) -> int:
        v = ctypes.c_uint32()
        _check(load().coop_query(self._h, ctypes.byref(v)))
        return v.value

    def current_m(self) -> int:
        v = ctypes.c_uint32()
        _check(load().coop_current_m(self._h, ctypes.byref(v)))
        return v.value

    def wait(self, *, trace_cap=0, level_cap=0, event_cap=0) -> RunStats:
        st, bufs = _stats_struct(trace_cap, level_cap, event_cap)
        rc = load().coop_wait(self._h, ctypes.byref(st))
        load().coop_destroy(self._h)
        self._h = None
        _check(rc)
        return _to_runstats(st, bufs)

    def close(self):
        """Synchronise and release the kernel's resources (idempotent)."""
        if getattr(self, "_h", None):
            load().coop_destroy(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------- device API (coop_device.cuh)
class DevHandle:
    """Control block of the device API (coop_dev_create); resource messages
    (demand / grant) may be posted from another thread while a call runs."""

    def __init__(self, *, max_wgs=0, init_wgs=0, policy=POLICY_NEVER, flags=0, seed=1, resize_prob=0.0,
                 kill_prob=0.0, fork_prob=0.0, max_fork=0, script=None, m_trace_cap=0, timeout_ns=0):
        lib = load()
        o = DevOpts(max_wgs=max_wgs, init_wgs=init_wgs, policy=policy, flags=flags, seed=seed,
                    resize_prob=resize_prob, kill_prob=kill_prob, fork_prob=fork_prob, max_fork=max_fork,
                    m_trace_cap=m_trace_cap, timeout_ns=timeout_ns)
        if script is not None:
            self._script = (ctypes.c_uint32 * len(script))(*script)
            o.script = self._script
            o.script_len = len(script)
        self.m_trace_cap = m_trace_cap
        h = _P()
        _check(lib.coop_dev_create(ctypes.byref(o), ctypes.byref(h)))
        self.h = h

    def demand(self, n: int):
        _check(load().coop_dev_demand(self.h, n))

    def grant(self, n: int):
        _check(load().coop_dev_grant(self.h, n))

    def _stats(self):
        st = DevStats()
        buf = None
        if self.m_trace_cap:
            buf = (ctypes.c_uint32 * self.m_trace_cap)()
            st.m_trace = buf
            st.m_trace_cap = self.m_trace_cap
        return st, buf

    @staticmethod
    def _to_dict(st, buf):
        d = {k: getattr(st, k) for k, _ in DevStats._fields_ if k not in ("m_trace", "m_trace_cap")}
        d["m_trace"] = list(buf[: min(st.episodes, len(buf))]) if buf is not None else []
        return d

    def close(self):
        if getattr(self, "h", None):
            load().coop_dev_destroy(self.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def fig4_bfs(h: DevHandle, g, source: int, levels_out=None, *, threads_per_wg=256):
    """Fig. 4 on the device API; returns (levels int32 tensor, stats dict)."""
    import torch
    csr, keep = _device_csr(g, False)
    if levels_out is None:
        levels_out = torch.empty(g.num_vertices, dtype=torch.int32, device=g.col_idx.device)
    st, buf = h._stats()
    _check(load().coop_fig4_bfs(h.h, ctypes.byref(csr), int(source), levels_out.data_ptr(), threads_per_wg,
                                ctypes.byref(st)))
    del keep
    return levels_out, DevHandle._to_dict(st, buf)


def pannotia(h: DevHandle, app: str, g, arg: int, out=None, *, threads_per_wg=256):
    """Table 1's color / mis / p-sssp on the device API (coop_color / coop_mis / coop_psssp).
    ``arg`` is the priority seed (color, mis) or the source (p-sssp).  Returns (output tensor,
    iterations, stats dict)."""
    import torch
    fn = {"color": "coop_color", "mis": "coop_mis", "psssp": "coop_psssp"}[app]
    csr, keep = _device_csr(g, app == "psssp")
    if out is None:
        out = torch.empty(g.num_vertices, dtype=torch.int32, device=g.col_idx.device)
    st, buf = h._stats()
    it = ctypes.c_uint32()
    _check(getattr(load(), fn)(h.h, ctypes.byref(csr), int(arg), out.data_ptr(), threads_per_wg, ctypes.byref(it),
                               ctypes.byref(st)))
    del keep
    return out, it.value, DevHandle._to_dict(st, buf)


def work_steal(h: DevHandle, *, seed: int, depth: int, max_fanout: int, fixed=False, rounds=0, queue_cap=0,
               threads_per_wg=256):
    """Cooperative work stealing (Fig. 2 + §3.2) over the implicit task tree R19.
    Returns (result dict {count, total, hist, steals}, stats dict)."""
    t = WsTree(seed=seed & 0xFFFFFFFFFFFFFFFF, depth=depth, max_fanout=max_fanout, fixed=1 if fixed else 0,
               rounds=rounds, queue_cap=queue_cap)
    r = WsResult()
    st, buf = h._stats()
    _check(load().coop_work_steal(h.h, ctypes.byref(t), threads_per_wg, ctypes.byref(r), ctypes.byref(st)))
    res = {"count": r.count, "total": r.total, "hist": list(r.hist[: depth + 1]), "steals": r.steals}
    return res, DevHandle._to_dict(st, buf)
