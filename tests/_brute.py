"""Independent brute-force / closed-form checkers used to PIN the oracle.

Nothing here shares code with oracle/ or the CUDA path: plain numpy over a
dense boolean adjacency matrix, written from the definitions in SURVEY.md
§8(c) (a triangle is a 3-set whose 3 pairs are edges; a 4-clique a 4-set
whose 6 pairs are edges; the graph is the simple undirected graph of the
input pairs without self-loops).
"""
from __future__ import annotations

import itertools
from math import comb

import numpy as np


def adjacency(src, dst):
    """Dense symmetric 0/1 matrix over the compacted vertex set (self-loops dropped)."""
    src = np.asarray(src, dtype=np.int64)
    dst = np.asarray(dst, dtype=np.int64)
    ids = np.unique(np.concatenate([src, dst]))
    u = np.searchsorted(ids, src)
    v = np.searchsorted(ids, dst)
    n = ids.size
    A = np.zeros((n, n), dtype=bool)
    A[u, v] = True
    A[v, u] = True
    np.fill_diagonal(A, False)
    return A


def triangles_brute(A) -> int:
    """Sum over pairs i<j adjacent of #k>j adjacent to both (each 3-set once)."""
    n = A.shape[0]
    t = 0
    for i in range(n):
        for j in np.nonzero(A[i, i + 1:])[0] + i + 1:
            t += int(np.count_nonzero(A[i, j + 1:] & A[j, j + 1:]))
    return t


def triangles_trace(A) -> int:
    """trace(A^3)/6 in float64 (exact while entries of A^2 * A stay < 2^53)."""
    F = A.astype(np.float64)
    return int(round(float(np.einsum("ij,ji->", F @ F, F)) / 6.0))


def four_cliques_brute(A) -> int:
    n = A.shape[0]
    k = 0
    for i in range(n):
        for j in np.nonzero(A[i, i + 1:])[0] + i + 1:
            cij = A[i] & A[j]
            for l in np.nonzero(cij[j + 1:])[0] + j + 1:
                k += int(np.count_nonzero(cij[l + 1:] & A[l, l + 1:]))
    return k


def four_cliques_subsets(A) -> int:
    """Literal definition: every 4-subset, all 6 pairs adjacent (tiny n only)."""
    n = A.shape[0]
    return sum(1 for q in itertools.combinations(range(n), 4)
               if all(A[a, b] for a, b in itertools.combinations(q, 2)))


def ordered_bindings(A, size: int) -> int:
    """Number of ORDERED tuples of distinct vertices forming a clique (the
    unpruned join result): equals size! times the clique count."""
    n = A.shape[0]
    c = 0
    for q in itertools.permutations(range(n), size):
        if all(A[q[a], q[b]] for a, b in itertools.combinations(range(size), 2)):
            c += 1
    return c


def elementary_symmetric(sizes, r: int) -> int:
    return sum(int(np.prod(c, dtype=object)) for c in itertools.combinations(list(sizes), r))


def kn_triangles(n: int) -> int:
    return comb(n, 3)


def kn_4cliques(n: int) -> int:
    return comb(n, 4)


def cliques_by_earliest_rank(src, dst, size: int) -> np.ndarray:
    """Literal definition of the rank-range counts: enumerate every `size`-set
    whose pairs are all edges (itertools, tiny n only), find its earliest vertex
    under the (degree, original id) order of SURVEY.md §8(c) step 3, and count
    it at that vertex's rank (its position in the ascending order).  Returns
    counts[rank] over the non-isolated vertices."""
    src = np.asarray(src, dtype=np.int64)
    dst = np.asarray(dst, dtype=np.int64)
    A = adjacency(src, dst)
    ids = np.unique(np.concatenate([src, dst]))
    deg = A.sum(axis=1)
    active = np.nonzero(deg)[0]
    order = sorted(active.tolist(), key=lambda i: (int(deg[i]), int(ids[i])))
    rank = {v: r for r, v in enumerate(order)}
    out = np.zeros(len(order), dtype=np.int64)
    for q in itertools.combinations(active.tolist(), size):
        if all(A[a, b] for a, b in itertools.combinations(q, 2)):
            out[min(rank[v] for v in q)] += 1
    return out
