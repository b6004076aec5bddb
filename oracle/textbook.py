"""O1 loader: ctypes binding of oracle/textbook.c (TEST INFRASTRUCTURE ONLY).

``bfs`` / ``dijkstra`` take a graphgen.CSR (any device; copied to host) and
return numpy arrays: int32 levels (-1 unreachable) / uint32 distances
(0xFFFFFFFF unreachable).  Definitions: see textbook.c header.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "textbook.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile textbook.c with gcc (plain -O2, no parallelism)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-o", _LIB, _SRC])
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        p = ctypes.c_void_p
        lib.oracle_bfs.argtypes = [ctypes.c_int64, p, p, ctypes.c_int64, p]
        lib.oracle_bfs.restype = ctypes.c_int
        lib.oracle_dijkstra.argtypes = [ctypes.c_int64, p, p, p, ctypes.c_int64, p]
        lib.oracle_dijkstra.restype = ctypes.c_int
        _lib = lib
    return _lib


def _host_arrays(g):
    ro = np.ascontiguousarray(g.row_offsets.cpu().numpy().astype(np.int64, copy=False))
    col = np.ascontiguousarray(g.col_idx.cpu().numpy().astype(np.int32, copy=False))
    return ro, col


def bfs_arrays(V: int, ro: np.ndarray, col: np.ndarray, source: int) -> np.ndarray:
    lib = _load()
    out = np.empty(V, dtype=np.int32)
    rc = lib.oracle_bfs(V, ro.ctypes.data, col.ctypes.data, int(source), out.ctypes.data)
    if rc != 0:
        raise ValueError(f"oracle_bfs failed rc={rc}")
    return out


def bfs(g, source: int) -> np.ndarray:
    ro, col = _host_arrays(g)
    return bfs_arrays(g.num_vertices, ro, col, source)


def dijkstra_arrays(V: int, ro: np.ndarray, col: np.ndarray, w: np.ndarray, source: int) -> np.ndarray:
    lib = _load()
    out = np.empty(V, dtype=np.uint32)
    rc = lib.oracle_dijkstra(V, ro.ctypes.data, col.ctypes.data, w.ctypes.data, int(source), out.ctypes.data)
    if rc != 0:
        raise ValueError(f"oracle_dijkstra failed rc={rc}")
    return out


def dijkstra(g, source: int) -> np.ndarray:
    ro, col = _host_arrays(g)
    w = np.ascontiguousarray(g.weights.cpu().numpy().astype(np.uint32))
    return dijkstra_arrays(g.num_vertices, ro, col, w, source)


def level_sizes(levels: np.ndarray) -> list[int]:
    """Per-level frontier sizes |{v : level[v] = L}| for L = 0..max."""
    lv = levels[levels >= 0]
    if lv.size == 0:
        return []
    return np.bincount(lv).tolist()
