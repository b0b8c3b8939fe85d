"""GPU parity for SURVEY.md §8(f) NEXT-4: node orderings as ingest variants
(PAPER.md:1065-1153).  An ordering changes the orientation (and so ranges,
out-degrees and run time) but never a count: every query must equal the oracle
under every ordering, and the oriented trie must hold each undirected edge once."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import paper_1503_02368_b200 as eh
import synth

pytestmark = pytest.mark.gpu

ORDERS = ["degree", "rev_degree", "random", "bfs", "hybrid", "shingle", "id"]


def _edges_from_export(row_ptr, col, orig):
    src = np.repeat(np.arange(orig.size), np.diff(row_ptr).astype(np.int64))
    u, v = orig[src].astype(np.uint64), orig[col].astype(np.uint64)
    lo, hi = np.minimum(u, v), np.maximum(u, v)
    return np.sort(lo << np.uint64(32) | hi)


@pytest.mark.parametrize("order", ORDERS)
@pytest.mark.parametrize("seed", range(3))
def test_counts_invariant_under_ordering(order, seed):
    src, dst = synth.rmat(11, 16, 1300 + seed) if seed < 2 else synth.er(500, 0.05, 1300 + seed)
    og = oracle.Graph(src, dst)
    try:
        with eh.Graph(src, dst, order=order) as g:
            assert g.count_triangles() == og.count_triangles()
            assert g.count_4cliques() == og.count_4cliques()
            assert g.count_lollipop() == og.count_lollipop()
            assert g.count_barbell() == og.count_barbell()
            assert g.count_triangles_unpruned() == og.count_triangles_unpruned()
            row_ptr, col, orig, _ = g.export()
            st = g.stats()
        assert st.m_undirected == og.m and st.n_active == og.n_vertices
        # every undirected edge exactly once, lists strictly increasing
        vid, _, off, adj = og.export()
        src_o = np.repeat(vid, np.diff(off).astype(np.int64)).astype(np.uint64)
        ref = np.sort(np.minimum(src_o, adj.astype(np.uint64)) << np.uint64(32) | np.maximum(src_o, adj.astype(np.uint64)))
        assert np.array_equal(_edges_from_export(row_ptr, col, orig), ref)
        for r in range(orig.size):
            seg = col[row_ptr[r]:row_ptr[r + 1]]
            assert np.all(np.diff(seg.astype(np.int64)) > 0) and np.all(seg > r)
    finally:
        og.close()


def test_orderings_change_the_orientation():
    src, dst = synth.rmat(12, 16, 77)
    d = {}
    for order in ORDERS:
        with eh.Graph(src, dst, order=order) as g:
            d[order] = g.stats().max_out_degree
            t = g.count_triangles()
    # degree ordering minimises the largest out-list; ascending degree maximises it
    assert d["degree"] < d["random"] < d["rev_degree"]
    assert t == oracle.count_triangles(src, dst)


@pytest.mark.parametrize("order", ORDERS)
def test_ordering_edge_cases(order):
    e = np.zeros(0, np.uint32)
    with eh.Graph(e, e, order=order) as g:
        assert g.count_triangles() == 0
    # several components (BFS leaves the others unreached), a hub, and K_40
    s1, d1 = synth.complete(40)
    s2, d2 = synth.star(500)
    s = np.concatenate([s1, s2 + 1000, np.array([5000], np.uint32)])
    d = np.concatenate([d1, d2 + 1000, np.array([5001], np.uint32)])
    with eh.Graph(s, d, order=order) as g:
        assert g.count_triangles() == 9880 and g.count_4cliques() == 91390


def test_id_order_orients_by_input_id():
    """EH_ORDER_ID: rank = position of the id among the active ids, edges low -> high id."""
    src, dst = synth.rmat(10, 8, 5)
    with eh.Graph(src, dst, order="id") as g:
        row_ptr, col, orig, _ = g.export()
        assert g.count_triangles() == oracle.count_triangles(src, dst)
    assert np.all(np.diff(orig.astype(np.int64)) > 0)  # ranks ascend by id
    act = np.unique(np.concatenate([src[src != dst], dst[src != dst]]))
    assert np.array_equal(orig, act)


def test_unknown_order_is_einval():
    with pytest.raises(KeyError):
        eh.Graph(np.array([0], np.uint32), np.array([1], np.uint32), order="nope")
