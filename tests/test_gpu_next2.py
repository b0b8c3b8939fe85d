"""GPU parity for SURVEY.md §8(f) NEXT-2: the triangle Generic-Join on the
UNPRUNED (symmetric) data, PAPER.md:1155-1236 -- CUDA path through the C ABI
vs the oracle's unpruned nest, bit-exact.  COUNT(*) binds ordered tuples, so
the result is 6T."""
from __future__ import annotations

import json
import os

import numpy as np
import pytest

import oracle
import paper_1503_02368_b200 as eh
import synth

pytestmark = pytest.mark.gpu


def _gpu(src, dst, **kw):
    with eh.Graph(src, dst, **kw) as g:
        return g.count_triangles_unpruned(), g.count_triangles(), g.symmetric_stats()


def _check(src, dst, **kw):
    u, t, st = _gpu(src, dst, **kw)
    og = oracle.Graph(src, dst)
    try:
        assert u == og.count_triangles_unpruned()
        assert u == 6 * t
        assert st.m_undirected == og.m and st.n_active == og.n_vertices
        _, deg, _, _ = og.export()
        assert st.max_out_degree == (int(deg.max()) if deg.size else 0)
    finally:
        og.close()
    return u


@pytest.mark.parametrize("n", list(range(0, 12)) + [65, 129, 300])
def test_kn(n):
    assert _gpu(*synth.complete(n))[0] == n * (n - 1) * (n - 2)


def test_k3000_above_2_32():
    assert _gpu(*synth.complete(3000), )[0] == 3000 * 2999 * 2998


@pytest.mark.parametrize("seed", range(12))
def test_random_er(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(2, 600))
    _check(*synth.er(n, float(rng.choice([0.002, 0.01, 0.05, 0.2])), seed))


@pytest.mark.parametrize("scale,ef,seed", [(s, ef, seed) for s in (6, 10, 13) for ef in (4, 16) for seed in range(2)])
def test_random_rmat(scale, ef, seed):
    _check(*synth.rmat(scale, ef, 7000 + 1000 * scale + 10 * ef + seed))


@pytest.mark.parametrize("seed", range(4))
def test_random_multigraph_with_noise(seed):
    src, dst = synth.random_graph(int(np.random.default_rng(seed).integers(3, 3000)), 20000, 90 + seed)
    _check(src, dst)


def test_empty_and_degenerate():
    e = np.zeros(0, np.uint32)
    assert _gpu(e, e)[0] == 0
    loops = np.arange(10, dtype=np.uint32)
    assert _gpu(loops, loops)[0] == 0
    assert _gpu(np.array([0, 1, 2], np.uint32), np.array([1, 2, 0], np.uint32))[0] == 6


def test_star_with_path_hub_unstaged():
    # the hub's full list (200k) exceeds every staging capacity: global sorted-list mode
    s, d = synth.star(200_000)
    leaves = np.arange(1, 200_001, dtype=np.uint32)
    s = np.concatenate([s, leaves[:-1]])
    d = np.concatenate([d, leaves[1:]])
    assert _gpu(s, d)[0] == 6 * 199_999


@pytest.mark.parametrize("kw", [dict(tau=256), dict(tau=2), dict(tau=1 << 20), dict(all_uint=True), dict(no_algo=True), dict(force_search=True),
                                dict(bin_small_max=2**32 - 1), dict(bin_large_min=1), dict(min_bitset_card=1)])
def test_layout_and_binning_invariance(kw):
    src, dst = synth.rmat(13, 16, 4243)
    assert _gpu(src, dst)[0] == _gpu(src, dst, **kw)[0]


@pytest.mark.parametrize("seed", range(2))
def test_unstaged_cta_path(seed, monkeypatch):
    monkeypatch.setenv("EH_TEST_TRI_XCAP", "128")
    _check(*synth.rmat(12, 16, 8100 + seed))


def test_rmat16_six_times_pruned():
    src, dst = synth.rmat(16, 16, 31)
    u, t, st = _gpu(src, dst)
    assert u == 6 * t and st.alg_bytes_tri > 0


@pytest.mark.parametrize("name", ["C1", "C2", "C4"])
def test_configs_vs_oracle_golden(name, golden_dir):
    gold = json.load(open(os.path.join(golden_dir, "configs_oracle.json")))["configs"][name]
    src, dst = synth.CONFIGS[name].generate()
    assert str(synth.checksum(src, dst)) == gold["checksum"]
    assert _gpu(src, dst)[0] == 6 * gold["triangles"]


# ------------------------------------------------------------ unpruned 4-clique --
def _k4u(src, dst, **kw):
    with eh.Graph(src, dst, **kw) as g:
        return g.count_4cliques_unpruned(), g.count_4cliques()


@pytest.mark.parametrize("n", [0, 3, 4, 5, 12, 64, 129, 200])
def test_k4_unpruned_kn(n):
    from math import comb
    assert _k4u(*synth.complete(n))[0] == 24 * comb(n, 4)


@pytest.mark.parametrize("seed", range(8))
def test_k4_unpruned_vs_oracle(seed):
    rng = np.random.default_rng(500 + seed)
    if seed % 2:
        src, dst = synth.rmat(int(rng.integers(6, 11)), 16, 500 + seed)
    else:
        src, dst = synth.er(int(rng.integers(20, 400)), float(rng.choice([0.02, 0.1, 0.3])), 500 + seed)
    u, k = _k4u(src, dst)
    og = oracle.Graph(src, dst)
    try:
        assert u == og.count_4cliques_unpruned() == 24 * k
    finally:
        og.close()


def test_k4_unpruned_hub_fallback():
    # complete graph K_1100: every list exceeds the 1024 bit-matrix limit (generic path)
    from math import comb
    assert _k4u(*synth.complete(1100))[0] == 24 * comb(1100, 4)


def _two_hubs_over_a_path(leaves: int):
    # hubs h1, h2 (adjacent) both joined to every leaf; a path over the leaves.  The
    # 4-cliques are exactly {h1, h2, l_i, l_i+1}: K4 = leaves - 1.  The row (h1, h2)
    # of the unpruned nest has P = all leaves.
    h1, h2 = leaves, leaves + 1
    lv = np.arange(leaves, dtype=np.uint32)
    src = np.concatenate([np.full(leaves, h1, np.uint32), np.full(leaves, h2, np.uint32), lv[:-1], [h1]])
    dst = np.concatenate([lv, lv, lv[1:], [h2]]).astype(np.uint32)
    return src.astype(np.uint32), dst


@pytest.mark.parametrize("leaves", [3000, 20000])
def test_k4_unpruned_hub_rows(leaves):
    # hub rows (|N(x)| > 1024) on the CTA-per-row kernel; with 20000 leaves the row
    # (h1, h2) has |P| = 20000, above the on-chip staging capacity (global scratch)
    src, dst = _two_hubs_over_a_path(leaves)
    u, k = _k4u(src, dst)
    assert k == leaves - 1 == oracle.count_4cliques(src, dst)
    assert u == 24 * (leaves - 1)


def test_k4_pruned_hub_rows():
    # pruned nest with |N+(x)| > 1024: K_1100's lowest-rank vertex has 1099 out-neighbours
    from math import comb
    with eh.Graph(*synth.complete(1100)) as g:
        assert g.stats().max_out_degree == 1099
        assert g.count_4cliques() == comb(1100, 4)


@pytest.mark.parametrize("kw", [dict(tau=2), dict(all_uint=True), dict(no_algo=True), dict(force_search=True), dict(bin_large_min=1)])
def test_k4_unpruned_invariance(kw):
    src, dst = synth.rmat(11, 16, 77)
    assert _k4u(src, dst)[0] == _k4u(src, dst, **kw)[0] == 24 * _k4u(src, dst)[1]
