"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This package holds no arithmetic of the method (no dedup, ordering, trie or
counting).  It draws edge lists only:

* ``rmat`` / ``er`` call the C generators in ``eh_synth.c`` (counter-based,
  parallel, bit-reproducible);
* ``CONFIGS`` are BASELINE.json's five workloads (C1..C5);
* the small structured families (complete, bipartite, r-partite, wheel, star,
  path) are used by the pins in ``tests/``.

Recipe: SURVEY.md §8(c) reading c19; DESIGN.md "Input recipe".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "eh_synth.c")
_SO = os.path.join(_HERE, "libehsynth.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile eh_synth.c into libehsynth.so (gcc, -O3, pthreads)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O3", "-march=x86-64-v2", "-fPIC", "-shared", "-pthread",
                               "-o", tmp, _SRC])
        os.replace(tmp, _SO)
    return _SO


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        u32p = ctypes.POINTER(ctypes.c_uint32)
        lib.eh_synth_rmat.argtypes = [ctypes.c_uint32, ctypes.c_uint64, ctypes.c_double, ctypes.c_double,
                                      ctypes.c_double, ctypes.c_uint64, ctypes.c_int, u32p, u32p, ctypes.c_int]
        lib.eh_synth_rmat.restype = ctypes.c_int
        lib.eh_synth_er.argtypes = [ctypes.c_uint32, ctypes.c_double, ctypes.c_uint64, u32p, u32p, ctypes.c_uint64]
        lib.eh_synth_er.restype = ctypes.c_uint64
        lib.eh_synth_checksum.argtypes = [u32p, u32p, ctypes.c_uint64]
        lib.eh_synth_checksum.restype = ctypes.c_uint64
        _lib = lib
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))


def rmat(scale: int, edge_factor: int, seed: int, a=0.57, b=0.19, c=0.19, scramble=True,
         threads: int | None = None, out: tuple[np.ndarray, np.ndarray] | None = None):
    """RMAT edge list: n_in = edge_factor * 2**scale uint32 tuples (src, dst).

    ``out`` may supply two preallocated uint32 arrays (e.g. pinned host memory).
    """
    n = int(edge_factor) << int(scale)
    if out is None:
        src = np.empty(n, dtype=np.uint32)
        dst = np.empty(n, dtype=np.uint32)
    else:
        src, dst = out
        assert src.dtype == np.uint32 and dst.dtype == np.uint32 and src.size >= n and dst.size >= n
    t = threads or os.cpu_count() or 1
    rc = _load().eh_synth_rmat(scale, n, a, b, c, seed, 1 if scramble else 0, _p(src), _p(dst), t)
    if rc != 0:
        raise ValueError("eh_synth_rmat: bad arguments")
    return src[:n], dst[:n]


def er(n: int, p: float, seed: int):
    """Erdos-Renyi G(n, p) edge list (each kept pair once, random direction)."""
    lib = _load()
    k = lib.eh_synth_er(n, p, seed, None, None, 0)
    src = np.empty(k, dtype=np.uint32)
    dst = np.empty(k, dtype=np.uint32)
    if k:
        lib.eh_synth_er(n, p, seed, _p(src), _p(dst), k)
    return src, dst


def checksum(src: np.ndarray, dst: np.ndarray) -> int:
    src = np.ascontiguousarray(src, dtype=np.uint32)
    dst = np.ascontiguousarray(dst, dtype=np.uint32)
    return int(_load().eh_synth_checksum(_p(src), _p(dst), src.size))


@dataclass(frozen=True)
class Config:
    name: str
    kind: str          # "er" | "rmat"
    query: str         # "triangles" | "4cliques"
    scale: int = 0
    edge_factor: int = 0
    n: int = 0
    p: float = 0.0
    seed: int = 0

    @property
    def n_input(self) -> int:
        return self.edge_factor << self.scale if self.kind == "rmat" else -1

    def generate(self, threads: int | None = None, out=None):
        if self.kind == "er":
            return er(self.n, self.p, self.seed)
        return rmat(self.scale, self.edge_factor, self.seed, threads=threads, out=out)


# BASELINE.json "configs", in order (SURVEY.md §8 shorthand C1..C5).
CONFIGS = {
    "C1": Config("C1", "er", "triangles", n=2000, p=0.005, seed=1),
    "C2": Config("C2", "rmat", "triangles", scale=18, edge_factor=16, seed=2),
    "C3": Config("C3", "rmat", "triangles", scale=22, edge_factor=16, seed=3),
    "C4": Config("C4", "rmat", "4cliques", scale=20, edge_factor=16, seed=4),
    "C5": Config("C5", "rmat", "triangles", scale=26, edge_factor=20, seed=5),
}


# ---------------------------------------------------------------- families --
def _pairs(u, v):
    return np.asarray(u, dtype=np.uint32), np.asarray(v, dtype=np.uint32)


def complete(n: int, offset: int = 0):
    """K_n on ids offset..offset+n-1, each pair once (i < j)."""
    i, j = np.triu_indices(n, 1)
    return _pairs(i + offset, j + offset)


def complete_multipartite(sizes, offset: int = 0):
    """Complete r-partite graph with the given part sizes."""
    part = np.repeat(np.arange(len(sizes)), sizes)
    i, j = np.triu_indices(len(part), 1)
    keep = part[i] != part[j]
    return _pairs(i[keep] + offset, j[keep] + offset)


def bipartite_random(n1: int, n2: int, p: float, seed: int):
    rng = np.random.default_rng(seed)
    m = rng.random((n1, n2)) < p
    i, j = np.nonzero(m)
    return _pairs(i, j + n1)


def wheel(k: int):
    """Wheel W_k: hub 0 plus a k-cycle on 1..k."""
    rim = np.arange(1, k + 1)
    nxt = np.roll(rim, -1)
    return _pairs(np.concatenate([np.zeros(k, np.int64), rim]), np.concatenate([rim, nxt]))


def star(k: int):
    """Star K_{1,k}: hub 0, leaves 1..k."""
    return _pairs(np.zeros(k, np.int64), np.arange(1, k + 1))


def random_graph(n: int, m: int, seed: int, id_space: int | None = None):
    """m random tuples over n vertices (duplicates / self-loops allowed),
    ids optionally spread over [0, id_space) by a seeded injective map."""
    rng = np.random.default_rng(seed)
    u = rng.integers(0, n, m)
    v = rng.integers(0, n, m)
    if id_space is not None:
        ids = np.sort(rng.choice(id_space, size=n, replace=False)).astype(np.uint64)
        rng.shuffle(ids)
        u, v = ids[u], ids[v]
    return _pairs(u, v)
