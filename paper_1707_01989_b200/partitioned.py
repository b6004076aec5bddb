"""1-D vertex-partitioned cooperative BFS across the GPUs of one node
(BASELINE.json configs[4]) -- host orchestration only.

Each rank owns a 32-aligned vertex range and holds every edge whose destination
it owns (graphgen.PartCSR).  The per-level frontier all-gather happens inside
libcoop's persistent kernel (coop_bfs_part): a rank stores its slice of the
next frontier bitmap straight into every peer's copy over NVLink and the
resizing barrier's serial section doubles as the cross-GPU barrier.  This
module only allocates the exchange buffers, shares them between ranks (CUDA IPC
handles all-gathered over torch.distributed, or plain pointers when several
ranks share one GPU in a test), and marshals the C structs.
"""
from __future__ import annotations

import ctypes
from typing import Optional, Sequence

import torch

from . import coop

MAX_RANKS = 8
HUB_DEGREE = 2048


CoopPart = coop.CoopPart


def _lib():
    return coop.load()


def hubs_of(part, hub_degree: int = HUB_DEGREE):
    """Static hubs: vertices whose LOCAL degree >= hub_degree, with the prefix
    sum of their local degrees (the edge space split evenly over all warps)."""
    ld = part.local_degrees()
    ids = torch.nonzero(ld >= hub_degree).flatten()
    pref = torch.zeros(ids.numel() + 1, dtype=torch.int64, device=ld.device)
    if ids.numel():
        pref[1:] = torch.cumsum(ld[ids], 0)
    return ids.to(torch.int32), pref


def exchange_handles(local: bytes, group=None) -> list[bytes]:
    """All-gather one opaque byte string per rank (IPC handles) over torch.distributed."""
    import torch.distributed as dist
    out: list = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, local, group=group)
    return out


class PartitionedBFS:
    """This rank's partition, exchange buffers and peer mapping.

    exchange="nvlink": the frontier slice is stored into every peer's bitmap by the
    kernel itself (coop_bfs_part; peers wired by connect_ipc / connect_local).
    exchange="nccl": north_star's data plane -- ncclAllGather of the slice on a comm
    stream ordered against the persistent kernel by stream memory operations
    (coop_bfs_part_nccl; communicator from connect_nccl)."""

    def __init__(self, part, device, hub_degree: int = HUB_DEGREE, exchange: str = "nvlink"):
        if exchange not in ("nvlink", "nccl"):
            raise ValueError(exchange)
        self.exchange = exchange
        self.comm = None
        self._own_comm = False
        self.part = part
        self.device = torch.device(device)
        self.V = part.num_vertices
        E = part.num_edges
        if E < (1 << 32):
            self.ro = part.row_offsets.to(self.device, torch.int32).contiguous()
            self.bits = 32
        else:
            self.ro = part.row_offsets.to(self.device, torch.int64).contiguous()
            self.bits = 64
        self.col = part.col_local.to(self.device, torch.int32).contiguous()
        import graphgen as gg
        rro, rcol = gg.part_rows(part)               # owned rows (bottom-up levels)
        self.rro = rro.to(self.device, torch.int32 if self.bits == 32 else torch.int64).contiguous()
        self.rcol = rcol.to(self.device).contiguous()
        del rro, rcol
        self.E_global = None                         # set by the caller (sum of num_edges over ranks)
        ids, pref = hubs_of(part, hub_degree)
        self.hub_ids = ids.to(self.device).contiguous()
        self.hub_pref = pref.to(self.device).contiguous()
        self.hub_degree = hub_degree
        # exchange buffers from cudaMalloc (shareable by CUDA IPC), zeroed once:
        # two frontier bitmaps of ceil(V/32) words (+16 B slack each) and the flag block
        lib = _lib()
        with torch.cuda.device(self.device):
            nw = (self.V + 31) // 32
            self.slice_words = (nw + part.nranks - 1) // part.nranks
            # NCCL: nranks uniform slices (in-place all-gather); NVLink: ceil(V/32) words + slack
            words = self.slice_words * part.nranks if exchange == "nccl" else nw
            self.nwb = (words * 4 + 16 + 255) // 256 * 256
            f = ctypes.c_void_p()
            coop._check(lib.coop_exchange_alloc(2 * self.nwb, ctypes.byref(f)))
            g = ctypes.c_void_p()
            coop._check(lib.coop_exchange_alloc(32 * MAX_RANKS, ctypes.byref(g)))
        self.F_ptr, self.flags_ptr = f.value, g.value
        self.levels = torch.empty(max(1, part.v_end - part.v_begin), dtype=torch.int32, device=self.device)
        self.peer_F = [[None, None] for _ in range(MAX_RANKS)]
        self.peer_flags = [None] * MAX_RANKS
        self._opened = []
        self.seq = 0

    # ---- peer wiring
    def connect_local(self, ranks: Sequence["PartitionedBFS"]):
        """All ranks share this process (and GPU): peers are plain device pointers."""
        for q, r in enumerate(ranks):
            self.peer_F[q] = [r.F_ptr, r.F_ptr + r.nwb]
            self.peer_flags[q] = r.flags_ptr

    def connect_ipc(self, group=None):
        """One process per GPU: all-gather CUDA IPC handles of F[0], F[1], flags."""
        lib = _lib()
        mine = b""
        for ptr in (self.F_ptr, self.flags_ptr):
            h = ctypes.create_string_buffer(64)
            coop._check(lib.coop_ipc_get_handle(ptr, h))
            mine += h.raw
        allh = exchange_handles(mine, group)
        nwb = self.nwb
        for q, blob in enumerate(allh):
            if q == self.part.rank:
                self.peer_F[q] = [self.F_ptr, self.F_ptr + nwb]
                self.peer_flags[q] = self.flags_ptr
                continue
            ptrs = []
            for k in range(2):
                p = ctypes.c_void_p()
                coop._check(lib.coop_ipc_open(blob[64 * k: 64 * (k + 1)], ctypes.byref(p)))
                self._opened.append(p.value)
                ptrs.append(p.value)
            self.peer_F[q] = [ptrs[0], ptrs[0] + nwb]
            self.peer_flags[q] = ptrs[1]

    def connect_nccl(self, comm_ptr: Optional[int] = None, group=None):
        """NCCL communicator of the partitioned BFS: torch's (``comm_ptr``, e.g.
        ProcessGroupNCCL._comm_ptr()) or a new one whose unique id rank 0 broadcasts
        over torch.distributed (``group``; a single-rank job needs no group)."""
        lib = _lib()
        if comm_ptr:
            self.comm = comm_ptr
            return
        uid = ctypes.create_string_buffer(128)
        if self.part.rank == 0:
            coop._check(lib.coop_nccl_get_unique_id(uid))
        if self.part.nranks > 1:
            import torch.distributed as dist
            obj = [uid.raw if self.part.rank == 0 else None]
            dist.broadcast_object_list(obj, src=0, group=group)
            uid = ctypes.create_string_buffer(obj[0], 128)
        c = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            coop._check(lib.coop_nccl_comm_init(self.part.nranks, uid, self.part.rank, ctypes.byref(c)))
        self.comm, self._own_comm = c.value, True

    def close(self):
        lib = _lib()
        if self.comm and self._own_comm:
            lib.coop_nccl_comm_destroy(ctypes.c_void_p(self.comm))
        self.comm = None
        for p in self._opened:
            lib.coop_ipc_close(ctypes.c_void_p(p))
        self._opened = []
        for p in (self.F_ptr, self.flags_ptr):
            if p:
                lib.coop_exchange_free(ctypes.c_void_p(p))
        self.F_ptr = self.flags_ptr = None

    # ---- calls
    def _struct(self, seq: int) -> CoopPart:
        s = CoopPart()
        s.num_vertices, s.v_begin, s.v_end = self.V, self.part.v_begin, self.part.v_end
        s.rank, s.nranks, s.seq = self.part.rank, self.part.nranks, seq & 0xFFFF
        s.row_offsets, s.offset_bits = self.ro.data_ptr(), self.bits
        s.col_local, s.num_edges = (self.col.data_ptr() if self.col.numel() else None), self.col.numel()
        s.num_hubs = self.hub_ids.numel()
        s.hub_ids = self.hub_ids.data_ptr() if s.num_hubs else None
        s.hub_prefix = self.hub_pref.data_ptr() if s.num_hubs else None
        s.hub_degree = self.hub_degree
        if self.exchange == "nccl":
            r = self.part.rank
            s.frontier[r][0], s.frontier[r][1] = self.F_ptr, self.F_ptr + self.nwb
        else:
            for q in range(self.part.nranks):
                s.frontier[q][0], s.frontier[q][1] = self.peer_F[q]
                s.flags[q] = self.peer_flags[q]
        s.rows_offsets = self.rro.data_ptr()
        s.rows_col = self.rcol.data_ptr() if self.rcol.numel() else None
        s.num_edges_global = int(self.E_global) if self.E_global else 0
        return s

    def launch(self, source: int, *, seq: Optional[int] = None, **opts):
        """Asynchronous: returns an opaque handle for wait()."""
        lib = _lib()
        if seq is None:
            self.seq += 1
            seq = self.seq
        self._s = self._struct(seq)
        self._o, self._k = coop.make_opts(**opts)
        h = ctypes.c_void_p()
        coop._check(lib.coop_bfs_part_launch(ctypes.byref(self._s), int(source), self.levels.data_ptr(),
                                             ctypes.byref(self._o), ctypes.byref(h)))
        return h

    def wait(self, h, level_cap: int = 0):
        lib = coop.load()
        st, bufs = coop._stats_struct(0, level_cap, 0)
        rc = lib.coop_wait(h, ctypes.byref(st))
        lib.coop_destroy(h)
        coop._check(rc)
        return coop._to_runstats(st, bufs)

    def run(self, source: int, *, level_cap: int = 0, **opts):
        """Blocking call of this rank (all ranks must call it with the same source)."""
        lib = _lib()
        self.seq += 1
        s = self._struct(self.seq)
        o, k = coop.make_opts(**opts)
        st, bufs = coop._stats_struct(0, level_cap, 0)
        if self.exchange == "nccl":
            if not self.comm:
                raise RuntimeError("connect_nccl() first")
            with torch.cuda.device(self.device):
                coop._check(lib.coop_bfs_part_nccl(ctypes.byref(s), int(source), self.levels.data_ptr(),
                                                   ctypes.c_void_p(self.comm), ctypes.byref(o), ctypes.byref(st)))
        else:
            coop._check(lib.coop_bfs_part(ctypes.byref(s), int(source), self.levels.data_ptr(), ctypes.byref(o),
                                          ctypes.byref(st)))
        return self.levels, coop._to_runstats(st, bufs)


def simulate_one_gpu(g, P: int, source: int, *, threads: int = 256, ctas_per_rank: Optional[int] = None,
                     device="cuda", parts=None, level_cap: int = 0, **opts):
    """P ranks on ONE GPU (test harness): P concurrent cooperative kernels, one
    per rank, each on its own stream and workspace, exchanging frontiers through
    plain device pointers -- the same kernel code as across NVLink."""
    import graphgen as gg
    if parts is None:
        parts = [PartitionedBFS(gg.partition(g, P, r), device) for r in range(P)]
    Eg = sum(pb.part.num_edges for pb in parts)
    for pb in parts:
        pb.connect_local(parts)
        pb.E_global = Eg
    info = coop.device_query(torch.device(device).index or 0, threads)
    n = ctas_per_rank or max(1, (info["max_coresident"] // P) // 2)
    streams = [torch.cuda.Stream(device=device) for _ in range(P)]
    torch.cuda.synchronize(device)
    seq = max(pb.seq for pb in parts) + 1
    hs = []
    for r, pb in enumerate(parts):
        pb.seq = seq
        hs.append(pb.launch(source, seq=seq, threads_per_wg=threads, max_wgs=n, workspace=r,
                            stream=streams[r].cuda_stream, **opts))
    stats = [pb.wait(h, level_cap) for pb, h in zip(parts, hs)]
    levels = torch.cat([pb.levels[: pb.part.v_end - pb.part.v_begin] for pb in parts])
    return levels, stats, parts


class PartitionedSSSP(PartitionedBFS):
    """This rank's share of the partitioned SSSP (coop_sssp_part): the BFS layout
    plus the local edge weights; the exchange buffers are (vertex, distance) inboxes
    of num_vertices uint64 each (two parities), shared like the BFS bitmaps."""

    def __init__(self, part, device):
        if part.weights is None:
            raise ValueError("partitioned SSSP needs a weighted partition")
        self.part = part
        self.device = torch.device(device)
        self.exchange = "nvlink"
        self.comm = None
        self._own_comm = False
        self.V = part.num_vertices
        E = part.num_edges
        self.bits = 32 if E < (1 << 32) else 64
        self.ro = part.row_offsets.to(self.device, torch.int32 if self.bits == 32 else torch.int64).contiguous()
        self.col = part.col_local.to(self.device, torch.int32).contiguous()
        self.w = part.weights.to(self.device, torch.int32).contiguous()
        self.rro = self.ro[:1]
        self.rcol = self.col[:0]
        self.E_global = None
        self.hub_ids = torch.zeros(0, dtype=torch.int32, device=self.device)
        self.hub_pref = torch.zeros(1, dtype=torch.int64, device=self.device)
        self.hub_degree = 0
        lib = _lib()
        with torch.cuda.device(self.device):
            self.nwb = (8 * self.V + 16 + 255) // 256 * 256
            f = ctypes.c_void_p()
            coop._check(lib.coop_exchange_alloc(2 * self.nwb, ctypes.byref(f)))
            g = ctypes.c_void_p()
            coop._check(lib.coop_exchange_alloc(32 * MAX_RANKS, ctypes.byref(g)))
        self.F_ptr, self.flags_ptr = f.value, g.value
        self.levels = torch.empty(max(1, part.v_end - part.v_begin), dtype=torch.int32, device=self.device)
        self.peer_F = [[None, None] for _ in range(MAX_RANKS)]
        self.peer_flags = [None] * MAX_RANKS
        self._opened = []
        self.seq = 0

    def launch(self, source: int, *, seq: Optional[int] = None, **opts):
        lib = _lib()
        if seq is None:
            self.seq += 1
            seq = self.seq
        self._s = self._struct(seq)
        self._o, self._k = coop.make_opts(**opts)
        h = ctypes.c_void_p()
        coop._check(lib.coop_sssp_part_launch(ctypes.byref(self._s), self.w.data_ptr() if self.w.numel() else None,
                                              int(source), self.levels.data_ptr(), ctypes.byref(self._o),
                                              ctypes.byref(h)))
        return h

    def run(self, source: int, *, level_cap: int = 0, **opts):
        lib = _lib()
        self.seq += 1
        s = self._struct(self.seq)
        o, k = coop.make_opts(**opts)
        st, bufs = coop._stats_struct(0, level_cap, 0)
        coop._check(lib.coop_sssp_part(ctypes.byref(s), self.w.data_ptr() if self.w.numel() else None, int(source),
                                       self.levels.data_ptr(), ctypes.byref(o), ctypes.byref(st)))
        return self.levels, coop._to_runstats(st, bufs)


def simulate_one_gpu_sssp(g, P: int, source: int, *, threads: int = 256, ctas_per_rank: int = 16,
                          device="cuda", parts=None, level_cap: int = 0, **opts):
    """P SSSP ranks on ONE GPU (test harness), as simulate_one_gpu for BFS."""
    import graphgen as gg
    if parts is None:
        parts = [PartitionedSSSP(gg.partition(g, P, r), device) for r in range(P)]
    for pb in parts:
        pb.connect_local(parts)
    streams = [torch.cuda.Stream(device=device) for _ in range(P)]
    torch.cuda.synchronize(device)
    seq = max(pb.seq for pb in parts) + 1
    hs = []
    for r, pb in enumerate(parts):
        pb.seq = seq
        hs.append(pb.launch(source, seq=seq, threads_per_wg=threads, max_wgs=ctas_per_rank, workspace=r,
                            stream=streams[r].cuda_stream, **opts))
    stats = [pb.wait(h, level_cap) for pb, h in zip(parts, hs)]
    dist = torch.cat([pb.levels[: pb.part.v_end - pb.part.v_begin] for pb in parts])
    return dist, stats, parts
