"""Pins of the CPU oracle against what the paper and mathematics fix (-m "not gpu").

Each test checks oracle/ against something other than itself: brute-force
enumeration, trace(A^3)/6, closed forms (K_n: PAPER.md:157-160, the AGM-tight
instance), complete r-partite e3/e4, bipartite zeros, wheels, hand-traced
worked examples (tests/golden/), a scipy.sparse library computation and
invariances under the input noise the paper's ingest removes (PAPER.md:284
"sets of distinct values", PAPER.md:799-800 pruning).
"""
from __future__ import annotations

import json
import os
from math import comb

import numpy as np
import pytest

import oracle
import synth
from tests import _brute as B


def _tri(src, dst, threads=4):
    return oracle.count_triangles(src, dst, threads)


def _k4(src, dst, threads=4):
    return oracle.count_4cliques(src, dst, threads)


# ------------------------------------------------------------ golden files --
def test_w1_worked_example(golden_dir):
    w = json.load(open(os.path.join(golden_dir, "w1_worked_example.json")))
    g = oracle.Graph(w["src"], w["dst"])
    assert g.m == w["m"] and g.n_vertices == w["n_vertices"]
    vid, deg, off, adj = g.export()
    for i, v in enumerate(vid):
        assert deg[i] == w["degrees"][str(v)]
        assert sorted(adj[off[i]:off[i + 1]].tolist()) == w["oriented_out"][str(v)]
    assert g.count_triangles(1) == w["triangles"]
    assert g.count_4cliques(1) == w["four_cliques"]


def test_w2_k5(golden_dir):
    w = json.load(open(os.path.join(golden_dir, "w2_k5.json")))
    assert _tri(w["src"], w["dst"]) == w["triangles"]
    assert _k4(w["src"], w["dst"]) == w["four_cliques"]


def test_w3_intersect(golden_dir):
    w = json.load(open(os.path.join(golden_dir, "w3_intersect.json")))
    for c in w["cases"]:
        b = list(range(0, 256)) if c["b"] == "range(0,256)" else c["b"]
        assert oracle.intersect(c["a"], b).tolist() == c["out"]


# ------------------------------------------------------------ brute force --
@pytest.mark.parametrize("seed", range(12))
def test_triangles_and_k4_vs_brute_force(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(5, 45))
    m = int(rng.integers(0, n * n // 2))
    src, dst = synth.random_graph(n, m, seed)
    A = B.adjacency(src, dst)
    assert _tri(src, dst) == B.triangles_brute(A) == B.triangles_trace(A)
    assert _k4(src, dst) == B.four_cliques_brute(A)


def test_k4_brute_matches_literal_subsets():
    # the faster brute force itself checked against the literal 4-subset definition
    for seed in range(4):
        src, dst = synth.random_graph(16, 70, 100 + seed)
        A = B.adjacency(src, dst)
        assert B.four_cliques_brute(A) == B.four_cliques_subsets(A) == _k4(src, dst)


@pytest.mark.parametrize("seed", range(3))
def test_rmat_small_vs_brute_force(seed):
    src, dst = synth.rmat(8, 8, 50 + seed)          # skewed, duplicates, self-loops
    A = B.adjacency(src, dst)
    assert _tri(src, dst) == B.triangles_brute(A) == B.triangles_trace(A)
    assert _k4(src, dst) == B.four_cliques_brute(A)


def test_unpruned_join_multiples():
    # symmetric (unpruned) data gives a multiple of the pruned result:
    # ordered bindings = 3! T and 4! K4
    src, dst = synth.random_graph(10, 35, 7)
    A = B.adjacency(src, dst)
    assert B.ordered_bindings(A, 3) == 6 * _tri(src, dst)
    assert B.ordered_bindings(A, 4) == 24 * _k4(src, dst)


# -------------------------------------------------------------- trace(A^3) --
def test_c1_triangles_trace():
    """C1 (ER n=2000, p=0.005, seed 1) pinned exactly by trace(A^3)/6."""
    src, dst = synth.CONFIGS["C1"].generate()
    A = B.adjacency(src, dst)
    assert _tri(src, dst) == B.triangles_trace(A)


@pytest.mark.parametrize("p", [0.01, 0.05, 0.2])
def test_er_trace(p):
    src, dst = synth.er(400, p, 11)
    A = B.adjacency(src, dst)
    assert _tri(src, dst) == B.triangles_trace(A)


def test_rmat_scipy_sparse():
    """Library routine: T = sum(U o (U @ U)) with U the id-ordered upper triangle
    (any strict order counts each triangle once)."""
    sp = pytest.importorskip("scipy.sparse")
    src, dst = synth.rmat(13, 16, 9)
    s = src.astype(np.int64)
    d = dst.astype(np.int64)
    keep = s != d
    lo = np.minimum(s[keep], d[keep])
    hi = np.maximum(s[keep], d[keep])
    n = int(max(s.max(), d.max())) + 1
    U = sp.csr_matrix((np.ones(lo.size, dtype=np.int64), (lo, hi)), shape=(n, n))
    U.data[:] = 1
    U.sum_duplicates()
    U.data[:] = 1
    T = int((U.multiply(U @ U)).sum())
    assert _tri(src, dst) == T


# ----------------------------------------------------------- closed forms --
@pytest.mark.parametrize("n", list(range(0, 21)) + [64, 200])
def test_kn_closed_form(n):
    src, dst = synth.complete(n)
    assert _tri(src, dst) == comb(n, 3)
    if n <= 64:
        assert _k4(src, dst) == comb(n, 4)


def test_k3000_triangles_above_2_32():
    src, dst = synth.complete(3000)
    t = _tri(src, dst, threads=oracle.default_threads())
    assert t == comb(3000, 3) == 4_495_501_000 and t > 2**32


def test_k600_four_cliques_above_2_32():
    src, dst = synth.complete(600)
    k = _k4(src, dst, threads=oracle.default_threads())
    assert k == comb(600, 4) == 5_346_164_850 and k > 2**32


@pytest.mark.parametrize("sizes", [(3, 4), (5, 5, 5), (2, 3, 4, 5), (1, 1, 1, 1, 1), (7, 1, 3, 2, 6)])
def test_complete_multipartite(sizes):
    src, dst = synth.complete_multipartite(sizes)
    assert _tri(src, dst) == B.elementary_symmetric(sizes, 3)
    assert _k4(src, dst) == B.elementary_symmetric(sizes, 4)


@pytest.mark.parametrize("seed", range(4))
def test_bipartite_zero(seed):
    src, dst = synth.bipartite_random(30 + seed, 40, 0.3, seed)
    assert _tri(src, dst) == 0 and _k4(src, dst) == 0
    src, dst = synth.complete_multipartite((20, 25))
    assert _tri(src, dst) == 0 and _k4(src, dst) == 0


@pytest.mark.parametrize("k", [4, 5, 6, 17, 100])
def test_wheel(k):
    src, dst = synth.wheel(k)
    assert _tri(src, dst) == k
    assert _k4(src, dst) == 0


def test_wheel3_is_k4():
    src, dst = synth.wheel(3)
    assert _tri(src, dst) == 4 and _k4(src, dst) == 1


# ------------------------------------------------------------ invariances --
def _perturb(src, dst, rng):
    """Random injective relabel into the full u32 space (0xFFFFFFFF included),
    random direction flips, duplicates and self-loops."""
    ids = np.unique(np.concatenate([src, dst]))
    new = rng.choice(2**32 - 1, size=ids.size, replace=False).astype(np.uint64)
    new[0] = 2**32 - 1
    rng.shuffle(new)
    s = new[np.searchsorted(ids, src)]
    d = new[np.searchsorted(ids, dst)]
    flip = rng.random(s.size) < 0.5
    s, d = np.where(flip, d, s), np.where(flip, s, d)
    dup = rng.integers(0, s.size, s.size // 3 + 1)
    loops = rng.choice(new, 10)
    s = np.concatenate([s, d[dup], loops])
    d = np.concatenate([d, s[dup], loops])
    p = rng.permutation(s.size)
    return s[p].astype(np.uint32), d[p].astype(np.uint32)


@pytest.mark.parametrize("seed", range(5))
def test_invariance_relabel_flip_dup_loops(seed):
    rng = np.random.default_rng(seed)
    src, dst = synth.rmat(10, 8, seed)
    s2, d2 = _perturb(src, dst, rng)
    assert _tri(src, dst) == _tri(s2, d2)
    assert _k4(src, dst) == _k4(s2, d2)


def test_disjoint_union_additive():
    a = synth.rmat(9, 8, 1)
    b = synth.rmat(9, 8, 2)
    off = np.uint32(1 << 20)
    s = np.concatenate([a[0], b[0] + off])
    d = np.concatenate([a[1], b[1] + off])
    assert _tri(s, d) == _tri(*a) + _tri(*b)
    assert _k4(s, d) == _k4(*a) + _k4(*b)


def test_thread_count_invariance():
    src, dst = synth.rmat(12, 16, 3)
    g = oracle.Graph(src, dst)
    t = {g.count_triangles(th) for th in (1, 2, 3, 8)}
    k = {g.count_4cliques(th) for th in (1, 2, 8)}
    assert len(t) == 1 and len(k) == 1


def test_k4_equals_sum_of_triangles_in_out_neighbourhoods():
    """K4 = sum_x T(G[N+(x)]): every 4-clique has a unique earliest vertex x and
    its other three vertices form a triangle inside N+(x)."""
    src, dst = synth.rmat(10, 12, 21)
    g = oracle.Graph(src, dst)
    vid, deg, off, adj = g.export()
    s_all, d_all = np.concatenate([src, dst]), np.concatenate([dst, src])
    total = 0
    for i in range(vid.size):
        nb = adj[off[i]:off[i + 1]]
        if nb.size < 3:
            continue
        inside = np.isin(s_all, nb) & np.isin(d_all, nb)
        total += _tri(s_all[inside], d_all[inside], threads=1)
    assert total == g.count_4cliques(4)


# --------------------------------------------------------------- ingest --
def test_ingest_structure():
    src, dst = synth.rmat(12, 16, 5)
    g = oracle.Graph(src, dst)
    vid, deg, off, adj = g.export()
    s = src.astype(np.int64); d = dst.astype(np.int64)
    keep = s != d
    pairs = np.unique(np.minimum(s, d)[keep] * 2**32 + np.maximum(s, d)[keep])
    assert g.m == pairs.size
    assert int(deg.sum()) == 2 * g.m
    assert int(off[-1]) == g.m
    pos = {int(v): i for i, v in enumerate(vid)}
    key = lambda v: (int(deg[pos[v]]), v)
    for i in range(vid.size):
        nb = adj[off[i]:off[i + 1]]
        assert np.all(np.diff(nb.astype(np.int64)) > 0)
        for w in nb.tolist():
            assert key(int(vid[i])) < key(w)


# -------------------------------------------------------------- intersect --
def test_intersect_vs_numpy():
    rng = np.random.default_rng(0)
    for t in range(2000):
        na, nb = rng.integers(0, 300, 2)
        hi = int(rng.choice([10, 1000, 2**20, 2**32]))
        a = np.unique(rng.integers(0, hi, na, dtype=np.uint64)).astype(np.uint32)
        b = np.unique(rng.integers(0, hi, nb, dtype=np.uint64)).astype(np.uint32)
        np.testing.assert_array_equal(oracle.intersect(a, b), np.intersect1d(a, b))


def test_triangles_at_sums_to_total():
    src, dst = synth.rmat(10, 16, 8)
    g = oracle.Graph(src, dst)
    vid, *_ = g.export()
    assert sum(g.triangles_at(int(v)) for v in vid) == g.count_triangles(2)
    assert g.count_triangles_range(0, vid.size // 2, 2) + g.count_triangles_range(vid.size // 2, vid.size, 3) \
        == g.count_triangles(1)


# ------------------------------------------------- NEXT-1: Lollipop / Barbell --
def _ordered_triangles(A):
    n = A.shape[0]
    return [(x, y, z) for x in range(n) for y in range(n) for z in range(n) if A[x, y] and A[y, z] and A[x, z]]


@pytest.mark.parametrize("seed", range(6))
def test_per_vertex_triangles_and_lollipop_barbell_vs_literal_join(seed):
    """Literal evaluation of the paper's queries over the SYMMETRIC relation
    (PAPER.md:227, 234, 877-878): every satisfying ordered tuple counted."""
    import itertools
    rng = np.random.default_rng(seed)
    n = int(rng.integers(4, 11))
    src, dst = synth.random_graph(n, int(rng.integers(n, n * n)), seed)
    A = B.adjacency(src, dst)
    g = oracle.Graph(src, dst)
    vid, *_ = g.export()
    ids = np.unique(np.concatenate([src, dst]).astype(np.int64))  # adjacency() compacts ids the same way
    pos = {int(v): i for i, v in enumerate(ids)}
    t_brute = [sum(1 for a, b in itertools.combinations(range(A.shape[0]), 2)
                   if A[v, a] and A[v, b] and A[a, b]) for v in range(A.shape[0])]
    t = g.triangles_per_vertex()
    for i, v in enumerate(vid):
        assert t[i] == t_brute[pos[int(v)]]
    assert int(t.sum()) == 3 * g.count_triangles(1)
    m = A.shape[0]
    lolli = sum(1 for x, y, z, w in itertools.product(range(m), repeat=4)
                if A[x, y] and A[y, z] and A[x, z] and A[x, w])
    assert g.count_lollipop() == lolli
    tri = _ordered_triangles(A)
    xs = np.array([p[0] for p in tri], dtype=np.int64)
    barb = int(A[np.ix_(xs, xs)].sum()) if xs.size else 0
    assert g.count_barbell() == barb


@pytest.mark.parametrize("n", [3, 4, 7, 30])
def test_lollipop_barbell_closed_forms_kn(n):
    g = oracle.Graph(*synth.complete(n))
    t = comb(n - 1, 2)
    assert np.all(g.triangles_per_vertex() == t)
    assert g.count_lollipop() == n * 2 * t * (n - 1)
    assert g.count_barbell() == n * (n - 1) * (2 * t) ** 2


def test_barbell_exceeds_u64_is_exact():
    # K_1630: Barbell = n(n-1)(2 C(n-1,2))^2 = 1.012 * 2^64 -> needs the 128-bit result
    n = 1630
    g = oracle.Graph(*synth.complete(n))
    val = n * (n - 1) * (2 * comb(n - 1, 2)) ** 2
    assert val > 2**64 and g.count_barbell() == val


# ------------------------------------------------------ NEXT-2: unpruned nests --
@pytest.mark.parametrize("seed", range(8))
def test_unpruned_nests_vs_ordered_bindings(seed):
    """oracle_count_{triangles,4cliques}_unpruned (the Generic-Join on the
    symmetric data) against brute-force ordered bindings."""
    rng = np.random.default_rng(300 + seed)
    n = int(rng.integers(4, 14))
    src, dst = synth.random_graph(n, int(rng.integers(0, n * n)), 300 + seed)
    A = B.adjacency(src, dst)
    g = oracle.Graph(src, dst)
    try:
        assert g.count_triangles_unpruned(2) == B.ordered_bindings(A, 3)
        assert g.count_4cliques_unpruned(2) == B.ordered_bindings(A, 4)
    finally:
        g.close()


@pytest.mark.parametrize("p", [0.02, 0.1])
def test_unpruned_triangles_trace(p):
    src, dst = synth.er(300, p, 17)
    A = B.adjacency(src, dst).astype(np.int64)
    g = oracle.Graph(src, dst)
    try:
        assert g.count_triangles_unpruned() == int(np.trace(A @ A @ A))  # ordered closed walks of length 3
    finally:
        g.close()


@pytest.mark.parametrize("n", [0, 1, 2, 3, 4, 9, 40])
def test_unpruned_kn_closed_forms(n):
    g = oracle.Graph(*synth.complete(n))
    try:
        assert g.count_triangles_unpruned() == n * (n - 1) * (n - 2)  # 3! C(n, 3)
        assert g.count_4cliques_unpruned() == 24 * comb(n, 4)
    finally:
        g.close()


def test_unpruned_rmat_multiples():
    src, dst = synth.rmat(11, 16, 41)
    g = oracle.Graph(src, dst)
    try:
        assert g.count_triangles_unpruned() == 6 * g.count_triangles()
        assert g.count_4cliques_unpruned() == 24 * g.count_4cliques()
    finally:
        g.close()


# ------------------------------------------------------------ rank ranges --
def test_w1_rank_ranges(golden_dir):
    """W1 hand trace: the two triangles are counted at x = r1 and x = r2."""
    w = json.load(open(os.path.join(golden_dir, "w1_worked_example.json")))
    g = oracle.Graph(w["src"], w["dst"])
    n = g.n_vertices
    assert [g.count_triangles_rank_range(r, r + 1, 1) for r in range(n)] == w["triangles_by_rank"]
    assert [g.count_4cliques_rank_range(r, r + 1, 1) for r in range(n)] == w["four_cliques_by_rank"]
    assert g.rank_ids().tolist() == w["rank_ids"]
    g.close()


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 9, 17, 40])
def test_rank_ranges_kn_closed_form(n):
    """K_n: every degree is n-1, so rank r is the r-th smallest id and the cliques
    whose earliest vertex is rank r choose their other members among the n-1-r
    later ones: C(n-1-r, 2) triangles, C(n-1-r, 3) 4-cliques."""
    src, dst = synth.complete(n, offset=1000)
    g = oracle.Graph(src, dst)
    for r in range(n):
        assert g.count_triangles_rank_range(r, r + 1, 2) == comb(n - 1 - r, 2)
        assert g.count_4cliques_rank_range(r, r + 1, 2) == comb(n - 1 - r, 3)
    assert g.count_4cliques_rank_range(0, n, 3) == comb(n, 4)
    assert g.count_triangles_rank_range(n, n + 5, 3) == 0
    g.close()


@pytest.mark.parametrize("seed", range(8))
def test_rank_ranges_vs_literal_enumeration(seed):
    rng = np.random.default_rng(900 + seed)
    n = int(rng.integers(6, 22))
    src, dst = synth.random_graph(n, int(rng.integers(n, 4 * n)), 900 + seed, id_space=1 << 32)
    t_ref = B.cliques_by_earliest_rank(src, dst, 3)
    k_ref = B.cliques_by_earliest_rank(src, dst, 4)
    g = oracle.Graph(src, dst)
    nv = g.n_vertices
    assert nv == t_ref.size
    assert [g.count_triangles_rank_range(r, r + 1, 2) for r in range(nv)] == t_ref.tolist()
    assert [g.count_4cliques_rank_range(r, r + 1, 2) for r in range(nv)] == k_ref.tolist()
    cuts = sorted(set([0, nv] + rng.integers(0, nv + 1, 3).tolist()))
    assert sum(g.count_4cliques_rank_range(a, b, 3) for a, b in zip(cuts, cuts[1:])) == g.count_4cliques(3)
    assert sum(g.count_triangles_rank_range(a, b, 3) for a, b in zip(cuts, cuts[1:])) == g.count_triangles(3)
    g.close()
