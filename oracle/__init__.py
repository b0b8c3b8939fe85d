"""CPU oracle for the EmptyHeaded hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product package ``paper_1503_02368_b200`` never imports it and shares no code
with it (see eh_oracle.c's header for the algorithm and its citations).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "eh_oracle.c")
_SO = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with plain gcc -O2 (no vectorisation tricks)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-pthread", "-o", tmp, _SRC])
        os.replace(tmp, _SO)
    return _SO


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        u32p = ctypes.POINTER(ctypes.c_uint32)
        u64p = ctypes.POINTER(ctypes.c_uint64)
        vp = ctypes.c_void_p
        lib.oracle_build.argtypes = [u32p, u32p, ctypes.c_uint64]
        lib.oracle_build.restype = vp
        lib.oracle_free.argtypes = [vp]
        lib.oracle_free.restype = None
        for name in ("oracle_count_triangles", "oracle_count_4cliques"):
            f = getattr(lib, name)
            f.argtypes = [vp, ctypes.c_int]
            f.restype = ctypes.c_uint64
        for name in ("oracle_count_triangles_range", "oracle_count_4cliques_range",
                     "oracle_count_triangles_rank_range", "oracle_count_4cliques_rank_range"):
            f = getattr(lib, name)
            f.argtypes = [vp, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int]
            f.restype = ctypes.c_uint64
        for name in ("oracle_count_triangles_unpruned", "oracle_count_4cliques_unpruned"):
            f = getattr(lib, name)
            f.argtypes = [vp, ctypes.c_int]
            f.restype = ctypes.c_uint64
        lib.oracle_rank_ids.argtypes = [vp, u32p]
        lib.oracle_rank_ids.restype = ctypes.c_int
        lib.oracle_triangles_at.argtypes = [vp, ctypes.c_uint32]
        lib.oracle_triangles_at.restype = ctypes.c_uint64
        lib.oracle_intersect.argtypes = [u32p, ctypes.c_uint64, u32p, ctypes.c_uint64, u32p]
        lib.oracle_intersect.restype = ctypes.c_int64
        lib.oracle_triangles_per_vertex.argtypes = [vp, u64p]
        lib.oracle_triangles_per_vertex.restype = None
        for name in ("oracle_count_lollipop", "oracle_count_barbell"):
            f = getattr(lib, name)
            f.argtypes = [vp, u64p]
            f.restype = ctypes.c_int
        lib.oracle_stats.argtypes = [vp, u64p]
        lib.oracle_stats.restype = None
        lib.oracle_export.argtypes = [vp, u32p, u32p, u64p, u32p]
        lib.oracle_export.restype = None
        _lib = lib
    return _lib


def _u32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a), dtype=np.uint32)


def _p32(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))


def default_threads() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)


class Graph:
    """Oracle trie of an edge list (original-id space, degree-oriented)."""

    def __init__(self, src, dst):
        lib = _load()
        self._src = _u32(src)
        self._dst = _u32(dst)
        if self._src.shape != self._dst.shape:
            raise ValueError("src and dst differ in length")
        h = lib.oracle_build(_p32(self._src), _p32(self._dst), self._src.size)
        if not h:
            raise MemoryError("oracle_build failed")
        self._h = ctypes.c_void_p(h)
        del self._src, self._dst
        st = (ctypes.c_uint64 * 4)()
        lib.oracle_stats(self._h, st)
        self.n_input, self.m, self.n_vertices, self.max_out_degree = (int(v) for v in st)

    def close(self):
        if getattr(self, "_h", None):
            _load().oracle_free(self._h)
            self._h = None

    __del__ = close

    def count_triangles(self, threads: int | None = None) -> int:
        return int(_load().oracle_count_triangles(self._h, threads or default_threads()))

    def count_4cliques(self, threads: int | None = None) -> int:
        return int(_load().oracle_count_4cliques(self._h, threads or default_threads()))

    def count_triangles_range(self, x0: int, x1: int, threads: int | None = None) -> int:
        return int(_load().oracle_count_triangles_range(self._h, x0, x1, threads or default_threads()))

    def count_4cliques_range(self, x0: int, x1: int, threads: int | None = None) -> int:
        return int(_load().oracle_count_4cliques_range(self._h, x0, x1, threads or default_threads()))

    def _rank_range(self, fn, r0: int, r1: int, threads):
        r = int(fn(self._h, r0, r1, threads or default_threads()))
        if r == 2**64 - 1:
            raise MemoryError("oracle allocation failed")
        return r

    def count_triangles_rank_range(self, r0: int, r1: int, threads: int | None = None) -> int:
        """Triangles whose earliest vertex has a rank in [r0, r1) of the ascending
        (degree, original id) order (eh_oracle.c "Rank ranges")."""
        return self._rank_range(_load().oracle_count_triangles_rank_range, r0, r1, threads)

    def count_4cliques_rank_range(self, r0: int, r1: int, threads: int | None = None) -> int:
        """4-cliques whose earliest vertex has a rank in [r0, r1) (eh_oracle.c "Rank ranges")."""
        return self._rank_range(_load().oracle_count_4cliques_rank_range, r0, r1, threads)

    def rank_ids(self) -> np.ndarray:
        """Original id of every rank of the (degree, original id) order."""
        ids = np.empty(max(self.n_vertices, 1), np.uint32)
        if _load().oracle_rank_ids(self._h, _p32(ids)) != 0:
            raise MemoryError("oracle allocation failed")
        return ids[:self.n_vertices]

    def count_triangles_unpruned(self, threads: int | None = None) -> int:
        """NEXT-2: the triangle Generic-Join on the symmetric (unpruned) data = 6T."""
        r = int(_load().oracle_count_triangles_unpruned(self._h, threads or default_threads()))
        if r == 2**64 - 1:
            raise MemoryError("oracle allocation failed")
        return r

    def count_4cliques_unpruned(self, threads: int | None = None) -> int:
        """NEXT-2: the 4-clique Generic-Join on the symmetric (unpruned) data = 24 K4."""
        r = int(_load().oracle_count_4cliques_unpruned(self._h, threads or default_threads()))
        if r == 2**64 - 1:
            raise MemoryError("oracle allocation failed")
        return r

    def triangles_at(self, x: int) -> int:
        return int(_load().oracle_triangles_at(self._h, x))

    def triangles_per_vertex(self) -> np.ndarray:
        """t(v) = number of triangles containing v, for v = vid[i] (sorted original ids)."""
        t = np.empty(max(self.n_vertices, 1), np.uint64)
        _load().oracle_triangles_per_vertex(self._h, t.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)))
        return t[:self.n_vertices]

    def _count128(self, fn) -> int:
        out = (ctypes.c_uint64 * 2)()
        if fn(self._h, out) != 0:
            raise MemoryError("oracle allocation failed")
        return int(out[0]) | (int(out[1]) << 64)

    def count_lollipop(self) -> int:
        """COUNT(*) of Lollipop L3,1 on the undirected data."""
        return self._count128(_load().oracle_count_lollipop)

    def count_barbell(self) -> int:
        """COUNT(*) of Barbell B3,1 on the undirected data."""
        return self._count128(_load().oracle_count_barbell)

    def export(self, with_adj: bool = True):
        """(vid, deg, off, adj): sorted original ids, degrees, out-list offsets,
        out-neighbours (original ids, each list sorted by original id; None
        unless with_adj)."""
        nv, m = self.n_vertices, self.m
        vid = np.empty(nv, np.uint32)
        deg = np.empty(nv, np.uint32)
        off = np.empty(nv + 1, np.uint64)
        adj = np.empty(m, np.uint32) if with_adj else None
        _load().oracle_export(self._h, _p32(vid), _p32(deg),
                              off.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
                              _p32(adj) if with_adj else None)
        return vid, deg, off, adj


def count_triangles(src, dst, threads: int | None = None) -> int:
    g = Graph(src, dst)
    try:
        return g.count_triangles(threads)
    finally:
        g.close()


def count_4cliques(src, dst, threads: int | None = None) -> int:
    g = Graph(src, dst)
    try:
        return g.count_4cliques(threads)
    finally:
        g.close()


def intersect(a, b) -> np.ndarray:
    """Sorted-merge intersection (Table `lst:eh_operators`)."""
    a = _u32(a)
    b = _u32(b)
    out = np.empty(min(a.size, b.size), np.uint32)
    k = _load().oracle_intersect(_p32(a), a.size, _p32(b), b.size, _p32(out))
    return out[:k]
