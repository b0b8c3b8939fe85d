"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, bit-exact.

All counts are integers, so every comparison is exact equality (BASELINE.json
north_star: "GPU counts must match the oracle bit-exact").  Inputs are seeded
and synthetic (synth/), shaped like the paper's workloads.
"""
from __future__ import annotations

import json
import os
from math import comb

import numpy as np
import pytest

import oracle
import paper_1503_02368_b200 as eh
import synth

pytestmark = pytest.mark.gpu


def _gpu_counts(src, dst, k4=True, **kw):
    with eh.Graph(src, dst, **kw) as g:
        t = g.count_triangles()
        k = g.count_4cliques() if k4 else None
        return t, k, g.stats()


def _oracle(src, dst, k4=True):
    g = oracle.Graph(src, dst)
    try:
        return g.count_triangles(), (g.count_4cliques() if k4 else None), g
    finally:
        pass


def _check(src, dst, k4=True, **kw):
    t, k, st = _gpu_counts(src, dst, k4=k4, **kw)
    ot, ok, og = _oracle(src, dst, k4=k4)
    assert t == ot, (t, ot)
    if k4:
        assert k == ok, (k, ok)
    assert st.m_undirected == og.m and st.n_active == og.n_vertices and st.max_out_degree == og.max_out_degree
    og.close()
    return t, k


# ------------------------------------------------------------ golden / closed forms --
def test_golden_w1_w2(golden_dir):
    for name in ("w1_worked_example.json", "w2_k5.json"):
        w = json.load(open(os.path.join(golden_dir, name)))
        t, k, _ = _gpu_counts(w["src"], w["dst"])
        assert (t, k) == (w["triangles"], w["four_cliques"])


@pytest.mark.parametrize("n", list(range(0, 24)) + [64, 100, 257])
def test_kn(n):
    t, k, _ = _gpu_counts(*synth.complete(n))
    assert t == comb(n, 3) and k == comb(n, 4)


def test_k3000_triangles_and_k600_4cliques_above_2_32():
    t, _, _ = _gpu_counts(*synth.complete(3000), k4=False)
    assert t == comb(3000, 3) == 4_495_501_000
    with eh.Graph(*synth.complete(600)) as g:
        assert g.count_4cliques() == comb(600, 4) == 5_346_164_850


@pytest.mark.parametrize("sizes", [(3, 4), (5, 5, 5), (2, 3, 4, 5), (30, 40, 50), (7, 1, 3, 2, 6, 9)])
def test_multipartite(sizes):
    t, k, _ = _gpu_counts(*synth.complete_multipartite(sizes))
    assert t == sum(a * b * c for i, a in enumerate(sizes) for j, b in enumerate(sizes[i + 1:], i + 1)
                    for c in sizes[j + 1:])
    assert k == oracle.count_4cliques(*synth.complete_multipartite(sizes))


def test_bipartite_and_wheel():
    for seed in range(3):
        t, k, _ = _gpu_counts(*synth.bipartite_random(200, 300, 0.2, seed))
        assert t == 0 and k == 0
    for kk in (3, 4, 5, 50, 1000):
        t, k, _ = _gpu_counts(*synth.wheel(kk))
        assert t == (4 if kk == 3 else kk) and k == (1 if kk == 3 else 0)


# -------------------------------------------------------------------- random graphs --
@pytest.mark.parametrize("seed", range(40))
def test_random_er(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(2, 600))
    p = float(rng.choice([0.002, 0.01, 0.05, 0.2]))
    _check(*synth.er(n, p, seed))


@pytest.mark.parametrize("scale,ef,seed", [(s, ef, seed) for s in (6, 8, 10, 12, 14) for ef in (4, 16)
                                           for seed in range(4)])
def test_random_rmat(scale, ef, seed):
    _check(*synth.rmat(scale, ef, 1000 * scale + 10 * ef + seed))


@pytest.mark.parametrize("seed", range(20))
def test_random_multigraph_with_noise(seed):
    src, dst = synth.random_graph(int(np.random.default_rng(seed).integers(3, 3000)), 20000, seed)
    _check(src, dst)


# ---------------------------------------------------------------------- edge cases --
def test_empty_and_degenerate():
    e = np.zeros(0, np.uint32)
    assert _gpu_counts(e, e)[:2] == (0, 0)
    loops = np.arange(100, dtype=np.uint32)
    assert _gpu_counts(loops, loops)[:2] == (0, 0)
    assert _gpu_counts(np.array([5], np.uint32), np.array([9], np.uint32))[:2] == (0, 0)
    tri = (np.array([0, 1, 2], np.uint32), np.array([1, 2, 0], np.uint32))
    assert _gpu_counts(*tri)[:2] == (1, 0)


def test_ids_near_u32_max_dictionary_path():
    rng = np.random.default_rng(3)
    src, dst = synth.rmat(11, 8, 77)
    ids = np.unique(np.concatenate([src, dst]))
    new = rng.choice(2**32 - 1, size=ids.size, replace=False).astype(np.uint64)
    new[-1] = 2**32 - 1
    s = new[np.searchsorted(ids, src)].astype(np.uint32)
    d = new[np.searchsorted(ids, dst)].astype(np.uint32)
    assert _check(s, d) == _check(src, dst)


@pytest.mark.parametrize("seed", range(2))
def test_unstaged_cta_path(seed, monkeypatch):
    # EH_TEST_TRI_XCAP (test hook) lowers the triangle CTA kernel's staging capacity:
    # every |N+(x)| > 128 then reads N+(x) from global memory (sorted-list mode).
    monkeypatch.setenv("EH_TEST_TRI_XCAP", "128")
    _check(*synth.rmat(14, 16, 555 + seed), k4=False)
    a = 300
    assert _gpu_counts(*synth.complete_multipartite((a, a, a)), k4=False)[0] == a**3


def test_huge_star_and_hub():
    s, d = synth.star(200_000)
    assert _gpu_counts(s, d)[:2] == (0, 0)
    # star plus a path over the leaves: every path edge closes one triangle with the hub
    leaves = np.arange(1, 200_001, dtype=np.uint32)
    s = np.concatenate([s, leaves[:-1]])
    d = np.concatenate([d, leaves[1:]])
    assert _gpu_counts(s, d, k4=True)[:2] == (199_999, 0)


@pytest.mark.parametrize("stride", [256, 512, 1 << 12])
def test_constant_low_digits(stride):
    # every id a multiple of `stride`: the canonical keys' low 8 / 9 / 12 bits are
    # constant, so the first radix pass(es) are skipped as trivial and the fused
    # canonicalisation runs in a later pass (or, with one distinct key, alone)
    leaves = (np.arange(1, 301, dtype=np.uint32) * stride).astype(np.uint32)
    s = np.concatenate([np.zeros(300, np.uint32), leaves[:-1]])
    d = np.concatenate([leaves, leaves[1:]])
    _check(s, d)
    assert _gpu_counts(s, d)[:2] == (299, 0)
    one = np.full(1000, stride, np.uint32)  # one distinct edge, repeated: every pass trivial
    assert _gpu_counts(np.zeros(1000, np.uint32), one)[2].m_undirected == 1


@pytest.mark.parametrize("xcap", [None, "128"])
def test_wide_shape_tma_staging(monkeypatch, xcap):
    # EH_TEST_TRI_WIDE (test hook) runs the wide (> 2^24 ids) triangle kernels on a small
    # graph: N+(x) staged by TMA (cp.async.bulk + mbarrier) double buffering; with
    # EH_TEST_TRI_XCAP=128 the lists above 128 take the unstaged branch (mbarrier phase
    # completed without a copy)
    src, dst = synth.rmat(14, 16, 41)
    ref = oracle.count_triangles(src, dst)
    monkeypatch.setenv("EH_TEST_TRI_WIDE", "1")
    if xcap:
        monkeypatch.setenv("EH_TEST_TRI_XCAP", xcap)
    with eh.Graph(src, dst) as g:
        assert g.stats().max_out_degree > 128
        assert g.count_triangles() == ref


@pytest.mark.parametrize("mid", ["0", "135", "512", "4096"])
def test_wide_shape_mid_class(monkeypatch, mid):
    # wide shape: class-2 x with |N+(x)| <= EH_TEST_TRI_MID (default 512) run on 4-warp CTAs
    # beside the 16-warp CTAs of the rest; any boundary (none, both classes populated, all
    # mid) gives the oracle's count, and the rank-range counts still add up
    from math import comb
    src, dst = synth.rmat(14, 16, 41)
    ref = oracle.count_triangles(src, dst)
    monkeypatch.setenv("EH_TEST_TRI_WIDE", "1")
    monkeypatch.setenv("EH_TEST_TRI_MID", mid)
    with eh.Graph(src, dst) as g:
        st = g.stats()
        assert st.max_out_degree > 135
        assert g.count_triangles() == ref
        cut = st.n_active - 3000
        assert g.count_triangles_range(0, cut) + g.count_triangles_range(cut, st.n_active) == ref
    n = 700  # K_700: |N+(x)| = 699 .. 0, both classes at the default boundary
    iu = np.triu_indices(n, 1)
    with eh.Graph(iu[0].astype(np.uint32), iu[1].astype(np.uint32)) as g:
        assert g.count_triangles() == comb(n, 3)


@pytest.mark.parametrize("offset", [0, 1, 3])
def test_device_inputs_unaligned(offset):
    # device-resident inputs that start 4 / 12 bytes past an aligned address: the
    # id-range pass falls back from 128-bit to 32-bit loads; counts are unchanged
    import torch
    src, dst = synth.rmat(13, 16, 61)
    ts = torch.from_numpy(src.view(np.int32)).cuda()[offset:]
    td = torch.from_numpy(dst.view(np.int32)).cuda()[offset:]
    with eh.Graph(ts, td) as g:
        assert g.count_triangles() == oracle.count_triangles(src[offset:], dst[offset:])


def test_block_cache_reuse_across_streams():
    # the default allocation path caches large blocks (>= 4 MB) across loads; a block
    # released on one stream and reused on another must wait for the first stream's
    # work (event-ordered): alternate loads / counts between two streams and a
    # library-owned one, and free the handles in a different order than they were made
    import torch
    src, dst = synth.rmat(16, 16, 31)   # 1 M input edges: 8 MB key buffers
    ref = oracle.count_triangles(src, dst)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    live = []
    for r in range(6):
        st = (s1, s2, None)[r % 3]
        g = eh.Graph(src, dst, stream=st) if st is not None else eh.Graph(src, dst)
        assert g.count_triangles() == ref
        live.append(g)
        if len(live) == 2:
            live.pop(0).close()
    for g in live:
        g.close()


# ------------------------------------------------------------------ invariances (T5/T6) --
@pytest.mark.parametrize("kw", [dict(tau=256), dict(tau=2), dict(tau=1 << 20), dict(all_uint=True), dict(no_algo=True), dict(force_search=True), dict(block_layout=True),
                                dict(block_layout=True, tau=2), dict(block_layout=True, bin_large_min=1),
                                dict(min_bitset_card=1), dict(bin_small_max=2**32 - 1),
                                dict(bin_small_max=1, bin_large_min=1), dict(bin_small_max=1, bin_large_min=2**32 - 1),
                                dict(torch_allocator=True), dict(bin_thread_max=1), dict(bin_thread_max=2),
                                dict(bin_thread_max=16), dict(bin_thread_max=16, bin_small_max=4)])
def test_layout_and_binning_invariance(kw):
    src, dst = synth.rmat(13, 16, 5)
    base = _gpu_counts(src, dst)[:2]
    assert _gpu_counts(src, dst, **kw)[:2] == base


@pytest.mark.parametrize("mode", ["hash", "sort"])
@pytest.mark.parametrize("seed", range(3))
def test_dedup_ablation_paths(seed, mode, monkeypatch):
    """EH_TEST_DEDUP=hash (one global hash set) and EH_TEST_DEDUP=sort (the one-sweep
    radix sort of the canonical keys) instead of the bucketed on-chip dedup of
    dedup.cu -- same trie, same counts."""
    src, dst = synth.rmat(13, 16, 70 + seed)
    l0 = eh.launch_count()
    base = _gpu_counts(src, dst)
    l1 = eh.launch_count()
    monkeypatch.setenv("EH_TEST_DEDUP", mode)
    alt = _gpu_counts(src, dst)
    l2 = eh.launch_count()
    assert l2 - l1 != l1 - l0  # the hook is read on every load: another kernel sequence ran
    assert base[:2] == alt[:2] == (oracle.count_triangles(src, dst), oracle.count_4cliques(src, dst))
    assert base[2] == alt[2]


@pytest.mark.parametrize("seed", range(3))
def test_bucket_classes_with_duplicates(seed):
    """Buckets of every dedup class (shared-memory tables of the small and big CTAs,
    global tables above 36,000 pairs) with heavy duplication and both orientations of
    each pair: hubs whose pairs fill one bucket, plus RMAT background."""
    rng = np.random.default_rng(seed)
    bs, bd = synth.rmat(14, 8, 900 + seed)
    parts_s, parts_d = [bs], [bd]
    for hub, k, rep in ((3, 60_000, 3), (70_000, 12_000, 2), (5, 3_000, 4)):
        nb = rng.choice(1 << 17, size=k, replace=False).astype(np.uint32)
        nb = np.repeat(nb, rep)
        flip = rng.random(nb.size) < 0.5
        parts_s.append(np.where(flip, nb, hub).astype(np.uint32))
        parts_d.append(np.where(flip, hub, nb).astype(np.uint32))
    s = np.concatenate(parts_s)
    d = np.concatenate(parts_d)
    perm = rng.permutation(s.size)
    _check(s[perm], d[perm])


@pytest.mark.parametrize("env", [dict(EH_TEST_BKT_CHUNK_MB="1"), dict(EH_TEST_BKT_PART_ATOMIC="1"),
                                 dict(EH_TEST_BKT_PART_MATCH="1"), dict(EH_TEST_BKT_GHIST="1"),
                                 dict(EH_TEST_BKT_SHIFT="2"), dict(EH_TEST_BKT_SHIFT="-3", EH_TEST_BKT_CHUNK_MB="1")])
@pytest.mark.parametrize("offset", [0, 1])
def test_bucket_partition_variants(env, offset, monkeypatch):
    """The bucket partition of dedup.cu: cursors in shared memory from per-(chunk, CTA)
    histograms (default; EH_TEST_BKT_CHUNK_MB=1 makes several chunks, with ragged last chunk),
    global cursor atomics (plain / warp-matched), the global-atomic histogram, other bucket
    widths; 16-B aligned and unaligned device inputs (128-bit / scalar loads).  Same trie."""
    import torch
    src, dst = synth.rmat(16, 16, 8800)
    src, dst = src[:-3], dst[:-3]  # n % 4 != 0
    ref = (oracle.count_triangles(src[offset:], dst[offset:]), oracle.count_4cliques(src[offset:], dst[offset:]))
    ts = torch.from_numpy(src.view(np.int32)).cuda()[offset:]
    td = torch.from_numpy(dst.view(np.int32)).cuda()[offset:]
    with eh.Graph(ts, td) as g:
        base = (g.count_triangles(), g.count_4cliques(), g.stats().m_undirected)
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    with eh.Graph(ts, td) as g:
        alt = (g.count_triangles(), g.count_4cliques(), g.stats().m_undirected)
    assert base == alt and base[:2] == ref


def test_device_input_and_stream():
    import torch
    src, dst = synth.rmat(12, 16, 6)
    ts = torch.from_numpy(src.view(np.int32)).cuda()
    td = torch.from_numpy(dst.view(np.int32)).cuda()
    st = torch.cuda.Stream()
    with eh.Graph(ts, td, stream=st) as g:
        t = g.count_triangles()
    assert t == oracle.count_triangles(src, dst)


# ----------------------------------------------------------------------- ingest (T4) --
@pytest.mark.parametrize("seed", range(3))
def test_ingest_csr_matches_oracle(seed):
    src, dst = synth.rmat(12, 16, 40 + seed)
    with eh.Graph(src, dst) as g:
        row_ptr, col, orig, isb = g.export()
    og = oracle.Graph(src, dst)
    vid, deg, off, adj = og.export()
    n = vid.size
    assert orig.size == n and row_ptr[-1] == og.m
    # rank order = ascending (degree, original id)
    pos = np.searchsorted(vid, orig)
    assert np.array_equal(vid[pos], orig)
    key = deg[pos].astype(np.int64) * 2**32 + orig
    assert np.all(np.diff(key) > 0)
    for r in range(n):
        lst = col[row_ptr[r]:row_ptr[r + 1]]
        assert np.all(np.diff(lst.astype(np.int64)) > 0) and (lst.size == 0 or lst[0] > r)
        i = pos[r]
        assert np.array_equal(np.sort(orig[lst]), adj[off[i]:off[i + 1]])


# ---------------------------------------------------------------- configs C1..C4 --
@pytest.mark.parametrize("name", ["C1", "C2"])
def test_config_small(name):
    cfg = synth.CONFIGS[name]
    _check(*cfg.generate(), k4=(name == "C2"))


def test_config_c3_triangles():
    src, dst = synth.CONFIGS["C3"].generate()
    t, _, st = _gpu_counts(src, dst, k4=False)
    assert t == oracle.count_triangles(src, dst)


def test_config_c4_4cliques():
    src, dst = synth.CONFIGS["C4"].generate()
    with eh.Graph(src, dst) as g:
        k = g.count_4cliques()
    assert k == oracle.count_4cliques(src, dst) and k > 2**32


# ----------------------------------------------------------------------- intersect --
def test_intersect_golden(golden_dir):
    w = json.load(open(os.path.join(golden_dir, "w3_intersect.json")))
    for c in w["cases"]:
        b = list(range(0, 256)) if c["b"] == "range(0,256)" else c["b"]
        assert eh.intersect(np.array(c["a"], np.uint32), np.array(b, np.uint32)).tolist() == c["out"]


def test_intersect_random_vs_numpy():
    rng = np.random.default_rng(1)
    for t in range(1500):
        na, nb = (int(v) for v in rng.integers(0, 2000, 2))
        if t % 7 == 0:
            nb = int(rng.integers(0, 200000))
        hi = int(rng.choice([64, 4096, 2**20, 2**32]))
        a = np.unique(rng.integers(0, hi, na, dtype=np.uint64)).astype(np.uint32)
        b = np.unique(rng.integers(0, hi, nb, dtype=np.uint64)).astype(np.uint32)
        got = eh.intersect(a, b)
        np.testing.assert_array_equal(got, np.intersect1d(a, b))
        assert eh.intersect(b, a, count_only=True) == got.size


def test_intersect_device_and_errors():
    import torch
    a = torch.arange(0, 1000, 3, dtype=torch.int32, device="cuda")
    b = torch.arange(0, 1000, 5, dtype=torch.int32, device="cuda")
    out = eh.intersect(a, b)
    assert out.is_cuda and out.cpu().tolist() == list(range(0, 1000, 15))
    with pytest.raises(eh.EHError) as ei:
        eh.intersect(np.array([3, 2], np.uint32), np.array([1], np.uint32))
    assert ei.value.status == eh.EH_EUNSORTED
    with pytest.raises(eh.EHError):
        eh.intersect(np.array([2, 2], np.uint32), np.array([1], np.uint32))


# ------------------------------------------------------------ error paths (T8) --
def test_allocator_hook_failure_is_enomem():
    """An allocator hook that returns NULL makes eh_load_edges fail cleanly with EH_ENOMEM."""
    import ctypes
    from paper_1503_02368_b200 import eh as ehmod
    L = ehmod.lib()
    alloc = ehmod._ALLOC_FN(lambda size, stream, ctx: None)
    free = ehmod._FREE_FN(lambda p, stream, ctx: None)
    src, dst = synth.rmat(10, 8, 1)
    cfg = ehmod.EHConfig()
    cfg.dev_alloc = alloc
    cfg.dev_free = free
    h = L.eh_load_edges_ex(src.ctypes.data, dst.ctypes.data, src.size, ctypes.byref(cfg))
    assert h is None and L.eh_last_status() == eh.EH_ENOMEM
    # the library stays usable afterwards
    assert _gpu_counts(src, dst)[0] == oracle.count_triangles(src, dst)


def test_invalid_device_and_graph_handles():
    import ctypes
    from paper_1503_02368_b200 import eh as ehmod
    L = ehmod.lib()
    cfg = ehmod.EHConfig()
    cfg.flags = eh.EH_SET_DEVICE
    cfg.device = 4096
    src, dst = synth.rmat(8, 8, 1)
    assert L.eh_load_edges_ex(src.ctypes.data, dst.ctypes.data, src.size, ctypes.byref(cfg)) is None
    assert L.eh_last_status() == eh.EH_EINVAL
    with pytest.raises(ValueError):
        eh.Graph(src, dst[:-1])


def test_repeated_counts_and_many_handles():
    """A handle is immutable after load: repeated counts agree; handles are independent."""
    graphs = [eh.Graph(*synth.rmat(11, 8, s)) for s in range(6)]
    first = [g.count_triangles() for g in graphs]
    again = [g.count_triangles() for g in reversed(graphs)][::-1]
    assert first == again
    for g in graphs:
        g.close()


# ------------------------------------------------- NEXT-3 block-level layout --
@pytest.mark.parametrize("seed", range(8))
def test_block_layout_vs_oracle(seed):
    """EH_BLOCK_LAYOUT: composite sets (128-id blocks, bitset blocks when >= 4
    elements) for the triangle count -- same counts as the oracle."""
    rng = np.random.default_rng(900 + seed)
    if seed % 3 == 0:
        src, dst = synth.rmat(int(rng.integers(8, 15)), 16, 900 + seed)
    elif seed % 3 == 1:
        src, dst = synth.er(int(rng.integers(50, 800)), float(rng.choice([0.05, 0.3, 0.8])), 900 + seed)
    else:
        src, dst = synth.complete_multipartite(tuple(int(x) for x in rng.integers(1, 60, size=4)))
    t, k, _ = _gpu_counts(src, dst, k4=True, block_layout=True)
    assert t == oracle.count_triangles(src, dst)
    assert k == oracle.count_4cliques(src, dst)  # other queries keep the set-level layouts


@pytest.mark.parametrize("kw", [dict(), dict(bin_small_max=2**32 - 1), dict(bin_large_min=1)])
def test_block_layout_dense_and_hashed_x(kw, monkeypatch):
    # K_400: every block dense; EH_TEST_TRI_XCAP forces hashed / sorted x structures (bit-by-bit dense path)
    from math import comb
    assert _gpu_counts(*synth.complete(400), k4=False, block_layout=True, **kw)[0] == comb(400, 3)
    monkeypatch.setenv("EH_TEST_TRI_XCAP", "128")
    assert _gpu_counts(*synth.complete(400), k4=False, block_layout=True, **kw)[0] == comb(400, 3)
    src, dst = synth.rmat(12, 16, 4)
    assert _gpu_counts(src, dst, k4=False, block_layout=True, **kw)[0] == oracle.count_triangles(src, dst)
