"""Seeded synthetic inputs shared by the CUDA path and the CPU oracle.

This package is the ONLY code both sides share (task rule ③): it produces
graphs (simple, symmetric, unweighted — PAPER.md §2) and seeded
right-hand-side vectors.  It contains none of the method's arithmetic: no walk
counts, no matrix functions, no Krylov.

Large random generators (R-MAT, Barabási–Albert, grid + deletion + LCC) are
C++ (``csrc/graphgen.cpp``, OpenMP, counter-based RNG, bit-exact for any
thread count); small fixed graphs (karate, the paper's trap graph G_{l,m},
paths, stars, cycles, complete graphs) are edge lists simplified by the same
C++ routine.  The workload recipes (configs C1..C5) are in ``configs.py``.
"""
from __future__ import annotations

import ctypes
import hashlib
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_lib", "libgraphgen.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile libgraphgen.so in-tree (g++ -O3 -fopenmp)."""
    src = os.path.join(_HERE, "csrc", "graphgen.cpp")
    if (not force and os.path.exists(_LIB_PATH)
            and os.path.getmtime(_LIB_PATH) >= os.path.getmtime(src)):
        return _LIB_PATH
    os.makedirs(os.path.dirname(_LIB_PATH), exist_ok=True)
    tmp = _LIB_PATH + f".tmp{os.getpid()}"
    cmd = ["g++", "-O3", "-std=c++17", "-fopenmp", "-fPIC", "-shared", src, "-o", tmp]
    subprocess.check_call(cmd)
    os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB_PATH)
        i64, vp = ctypes.c_int64, ctypes.c_void_p
        lib.gg_last_error.restype = ctypes.c_char_p
        lib.gg_rmat.argtypes = [ctypes.c_int, i64, i64, ctypes.c_double, ctypes.c_double,
                                ctypes.c_double, ctypes.c_uint64, ctypes.c_uint64,
                                ctypes.POINTER(vp)]
        lib.gg_ba.argtypes = [i64, ctypes.c_int, ctypes.c_uint64, ctypes.POINTER(vp)]
        lib.gg_grid_lcc.argtypes = [i64, i64, ctypes.c_double, ctypes.c_uint64,
                                    ctypes.POINTER(vp)]
        lib.gg_from_edges.argtypes = [i64, i64, vp, vp, ctypes.POINTER(vp)]
        lib.gg_n.argtypes = [vp]
        lib.gg_n.restype = i64
        lib.gg_nnz.argtypes = [vp]
        lib.gg_nnz.restype = i64
        lib.gg_copy.argtypes = [vp, vp, vp]
        lib.gg_destroy.argtypes = [vp]
        lib.gg_set_threads.argtypes = [ctypes.c_int]
        _lib = lib
    return _lib


@dataclass
class Graph:
    """CSR pattern of a simple undirected graph: row_ptr int64[n+1], col_idx int32[2m]."""

    n: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    name: str = ""

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    @property
    def degrees(self) -> np.ndarray:
        return np.diff(self.row_ptr)

    def sha256(self) -> str:
        h = hashlib.sha256()
        h.update(np.int64(self.n).tobytes())
        h.update(np.ascontiguousarray(self.row_ptr, dtype=np.int64).tobytes())
        h.update(np.ascontiguousarray(self.col_idx, dtype=np.int32).tobytes())
        return h.hexdigest()

    def dense(self) -> np.ndarray:
        a = np.zeros((self.n, self.n))
        rows = np.repeat(np.arange(self.n), self.degrees)
        a[rows, self.col_idx] = 1.0
        return a


def _take(handle) -> tuple[int, np.ndarray, np.ndarray]:
    lib = _load()
    n = lib.gg_n(handle)
    nnz = lib.gg_nnz(handle)
    rp = np.empty(n + 1, dtype=np.int64)
    ci = np.empty(nnz, dtype=np.int32)
    lib.gg_copy(handle, rp.ctypes.data, ci.ctypes.data)
    lib.gg_destroy(handle)
    return n, rp, ci


def _check(rc):
    if rc != 0:
        raise RuntimeError("graphgen: " + _load().gg_last_error().decode())


def from_edges(n: int, edges, name: str = "") -> Graph:
    """Simple graph from an edge list: loops dropped, duplicates merged, symmetrized."""
    e = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    u = np.ascontiguousarray(e[:, 0])
    v = np.ascontiguousarray(e[:, 1])
    h = ctypes.c_void_p()
    _check(_load().gg_from_edges(n, len(u), u.ctypes.data, v.ctypes.data, ctypes.byref(h)))
    n2, rp, ci = _take(h)
    return Graph(n2, rp, ci, name)


def rmat(scale: int, n: int, m: int, a=0.57, b=0.19, c=0.19, seed=3003, perm_seed=7,
         name: str = "") -> Graph:
    h = ctypes.c_void_p()
    _check(_load().gg_rmat(scale, n, m, a, b, c, seed, perm_seed, ctypes.byref(h)))
    n2, rp, ci = _take(h)
    return Graph(n2, rp, ci, name or f"rmat(scale={scale},n={n},m={m},seed={seed})")


def barabasi_albert(n: int, m0: int, seed: int, name: str = "") -> Graph:
    h = ctypes.c_void_p()
    _check(_load().gg_ba(n, m0, seed, ctypes.byref(h)))
    n2, rp, ci = _take(h)
    return Graph(n2, rp, ci, name or f"ba(n={n},m0={m0},seed={seed})")


def grid_lcc(nx: int, ny: int, p_del: float, seed: int, name: str = "") -> Graph:
    h = ctypes.c_void_p()
    _check(_load().gg_grid_lcc(nx, ny, p_del, seed, ctypes.byref(h)))
    n2, rp, ci = _take(h)
    return Graph(n2, rp, ci, name or f"grid_lcc({nx}x{ny},p={p_del},seed={seed})")


# --- small fixed graphs ------------------------------------------------------

# Zachary karate club, 0-based, 78 undirected edges, node order of networkx
# karate_club_graph() with weights ignored (Fig. 4
# uses "Newman/karate").
KARATE_EDGES = (
    "0-1 0-2 0-3 0-4 0-5 0-6 0-7 0-8 0-10 0-11 0-12 0-13 0-17 0-19 0-21 0-31 1-2 1-3 1-7 "
    "1-13 1-17 1-19 1-21 1-30 2-3 2-7 2-8 2-9 2-13 2-27 2-28 2-32 3-7 3-12 3-13 4-6 4-10 5-6 "
    "5-10 5-16 6-16 8-30 8-32 8-33 9-33 13-33 14-32 14-33 15-32 15-33 18-32 18-33 19-33 20-32 "
    "20-33 22-32 22-33 23-25 23-27 23-29 23-32 23-33 24-25 24-27 24-31 25-31 26-29 26-33 27-33 "
    "28-31 28-33 29-32 29-33 30-32 30-33 31-32 31-33 32-33")


def karate() -> Graph:
    edges = [tuple(int(x) for x in e.split("-")) for e in KARATE_EDGES.split()]
    return from_edges(34, edges, "karate")


def trap_graph(l: int = 5, m: int = 8) -> Graph:
    """G_{l,m}: a path 1..l plus m leaves on the central path node.

    0-based ids: path nodes 0..l-1, leaves l..l+m-1 attached to node (l-1)//2.
    For l=5, m=8 this is the paper's G_{5,8} with node k <-> paper label k+1.
    """
    c = (l - 1) // 2
    edges = [(i, i + 1) for i in range(l - 1)] + [(c, l + j) for j in range(m)]
    return from_edges(l + m, edges, f"G_{l},{m}")


def path(n: int) -> Graph:
    return from_edges(n, [(i, i + 1) for i in range(n - 1)], f"P{n}")


def cycle(n: int) -> Graph:
    return from_edges(n, [(i, (i + 1) % n) for i in range(n)], f"C{n}")


def complete(n: int) -> Graph:
    return from_edges(n, [(i, j) for i in range(n) for j in range(i + 1, n)], f"K{n}")


def star(leaves: int) -> Graph:
    return from_edges(leaves + 1, [(0, j) for j in range(1, leaves + 1)], f"star({leaves})")


def grid(nx: int, ny: int) -> Graph:
    e = [(i * ny + j, i * ny + j + 1) for i in range(nx) for j in range(ny - 1)]
    e += [(i * ny + j, (i + 1) * ny + j) for i in range(nx - 1) for j in range(ny)]
    return from_edges(nx * ny, e, f"grid({nx}x{ny})")


def with_isolated(g: Graph, extra: int) -> Graph:
    """Append `extra` isolated nodes (degenerate rows: the R-MAT configs have ~40%)."""
    rp = np.concatenate([g.row_ptr, np.full(extra, g.row_ptr[-1], dtype=np.int64)])
    return Graph(g.n + extra, rp, g.col_idx.copy(), g.name + f"+{extra}iso")


# --- seeded vectors -------------------------------------------------------------

def vectors(n: int, b: int, seed: int) -> np.ndarray:
    """Right-hand sides: numpy default_rng(seed).standard_normal((n, b)), fp64, row-major."""
    return np.random.default_rng(seed).standard_normal((n, b))
