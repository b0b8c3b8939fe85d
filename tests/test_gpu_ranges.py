"""GPU parity of the rank-range counts (eh_count_triangles_range /
eh_count_4cliques_range), B_K4 (eh_alg_bytes_k4), and the API contracts added
with them (stream ordering of device inputs, the release of cached memory,
checked outputs).

Range counts are bit-exact with the oracle's rank ranges (eh_oracle.c "Rank
ranges", pinned in tests/test_oracle_pins.py) and add up over any partition
of [0, n_active) to the full count.
"""
from __future__ import annotations

from math import comb

import numpy as np
import pytest

import oracle
import paper_1503_02368_b200 as eh
import synth

pytestmark = pytest.mark.gpu


def _cuts(n, k, rng):
    return sorted(set([0, n] + rng.integers(0, n + 1, k).tolist()))


@pytest.mark.parametrize("seed", range(10))
def test_ranges_vs_oracle(seed):
    rng = np.random.default_rng(4000 + seed)
    kind = seed % 3
    if kind == 0:
        src, dst = synth.rmat(int(rng.integers(8, 15)), 16, 4000 + seed)
    elif kind == 1:
        src, dst = synth.er(int(rng.integers(50, 700)), float(rng.choice([0.02, 0.1, 0.4])), 4000 + seed)
    else:
        src, dst = synth.random_graph(int(rng.integers(5, 400)), 5000, 4000 + seed, id_space=1 << 32)
    og = oracle.Graph(src, dst)
    with eh.Graph(src, dst) as g:
        n = g.stats().n_active
        assert n == og.n_vertices
        assert np.array_equal(g.export()[2], og.rank_ids())  # same rank space
        cuts = _cuts(n, 5, rng)
        tri = [g.count_triangles_range(a, b) for a, b in zip(cuts, cuts[1:])]
        k4 = [g.count_4cliques_range(a, b) for a, b in zip(cuts, cuts[1:])]
        assert tri == [og.count_triangles_rank_range(a, b) for a, b in zip(cuts, cuts[1:])]
        assert k4 == [og.count_4cliques_rank_range(a, b) for a, b in zip(cuts, cuts[1:])]
        assert sum(tri) == g.count_triangles() and sum(k4) == g.count_4cliques()
        # the full counts after a restricted one: the work lists are restored
        assert g.count_triangles() == og.count_triangles() and g.count_4cliques() == og.count_4cliques()
    og.close()


def test_ranges_kn_closed_form_and_edges():
    n = 300
    with eh.Graph(*synth.complete(n, offset=7)) as g:
        for r in (0, 1, 57, 200, n - 4, n - 3, n - 1):
            assert g.count_triangles_range(r, r + 1) == comb(n - 1 - r, 2)
            assert g.count_4cliques_range(r, r + 1) == comb(n - 1 - r, 3)
        assert g.count_4cliques_range(0, 2**64 - 1) == comb(n, 4)  # r1 clamped to n_active
        assert g.count_triangles_range(5, 5) == 0 and g.count_triangles_range(9, 3) == 0
        assert g.count_4cliques_range(n, n + 10) == 0
    e = np.zeros(0, np.uint32)
    with eh.Graph(e, e) as g:
        assert g.count_triangles_range(0, 10) == 0 and g.count_4cliques_range(0, 10) == 0


@pytest.mark.parametrize("kw", [dict(bin_small_max=2**32 - 1), dict(bin_large_min=1), dict(block_layout=True),
                                dict(all_uint=True), dict(bin_thread_max=1), dict(bin_thread_max=16)])
def test_ranges_invariant_under_classes_and_layouts(kw):
    src, dst = synth.rmat(13, 16, 4100)
    og = oracle.Graph(src, dst)
    with eh.Graph(src, dst, **kw) as g:
        n = g.stats().n_active
        for a, b in ((0, n // 2), (n // 2, n - 100), (n - 100, n)):
            assert g.count_triangles_range(a, b) == og.count_triangles_rank_range(a, b)
            assert g.count_4cliques_range(a, b) == og.count_4cliques_rank_range(a, b)
    og.close()


def test_ranges_hub_rows_k4_big():
    # |N+(x)| > 1024 takes the CTA-per-row 4-clique kernel (k_k4_big): K_1100 ranks
    n = 1100
    with eh.Graph(*synth.complete(n)) as g:
        assert g.stats().max_out_degree == n - 1
        assert g.count_4cliques_range(0, 1) == comb(n - 1, 3)
        assert g.count_4cliques_range(1, 40) == sum(comb(n - 1 - r, 3) for r in range(1, 40))


def _bytes32(row_ptr, col):
    """bytes(N+(v)) at tau = 32: 4 x words spanned for a bitset
    (span < 32 |S|), else 4 |S| -- written from the definition, in numpy."""
    n = row_ptr.size - 1
    out = np.zeros(n, np.int64)
    for v in range(n):
        lst = col[row_ptr[v]:row_ptr[v + 1]].astype(np.int64)
        if lst.size == 0:
            continue
        span = lst[-1] - lst[0] + 1
        out[v] = 4 * ((lst[-1] >> 5) - (lst[0] >> 5) + 1) if span < 32 * lst.size else 4 * lst.size
    return out


@pytest.mark.parametrize("seed", range(3))
def test_alg_bytes_k4_definition(seed):
    src, dst = synth.rmat(10, 8, 4200 + seed)
    with eh.Graph(src, dst) as g:
        row_ptr, col, _, _ = g.export()
        b_tri = g.stats().alg_bytes_tri
        b_k4 = g.alg_bytes_k4()
        assert g.alg_bytes_k4() == b_k4  # cached
    by = _bytes32(row_ptr, col)
    n = row_ptr.size - 1
    nbr = [set(col[row_ptr[v]:row_ptr[v + 1]].tolist()) for v in range(n)]
    extra = 0
    for x in range(n):
        for y in nbr[x]:
            for z in nbr[x] & nbr[y]:
                extra += int(by[z])
    ys = int(sum(by[c] for c in col))
    assert b_tri == 8 * (n + 1) + int(by.sum()) + ys
    assert b_k4 == b_tri + extra


def test_device_inputs_ordered_on_current_stream():
    """Device inputs still being written on torch's current (side) stream when the
    graph is loaded without an explicit stream: the binding passes the current
    stream, so the load is ordered after the writes."""
    import torch
    src, dst = synth.rmat(14, 16, 4300)
    ref = oracle.count_triangles(src, dst)
    side = torch.cuda.Stream()
    h_s = torch.from_numpy(src.view(np.int32)).pin_memory()
    h_d = torch.from_numpy(dst.view(np.int32)).pin_memory()
    for _ in range(3):
        with torch.cuda.stream(side):
            torch.cuda._sleep(50_000_000)  # ~25 ms of GPU time before the inputs are written
            ts = torch.zeros(src.size, dtype=torch.int32, device="cuda")
            td = torch.zeros(dst.size, dtype=torch.int32, device="cuda")
            ts.copy_(h_s, non_blocking=True)
            td.copy_(h_d, non_blocking=True)
            with eh.Graph(ts, td) as g:
                assert g.count_triangles() == ref
        side.synchronize()


def test_library_owned_stream_orders_after_default_stream():
    """No stream and host-side stream=None paths: the library-owned stream is a
    blocking stream, ordered after the legacy default stream's pending writes."""
    import torch
    from paper_1503_02368_b200 import eh as ehmod
    import ctypes
    src, dst = synth.rmat(13, 16, 4301)
    ref = oracle.count_triangles(src, dst)
    h_s = torch.from_numpy(src.view(np.int32)).pin_memory()
    h_d = torch.from_numpy(dst.view(np.int32)).pin_memory()
    torch.cuda._sleep(50_000_000)  # on the default stream
    ts = torch.empty(src.size, dtype=torch.int32, device="cuda").copy_(h_s, non_blocking=True)
    td = torch.empty(dst.size, dtype=torch.int32, device="cuda").copy_(h_d, non_blocking=True)
    L = ehmod.lib()
    cfg = ehmod.EHConfig()
    cfg.flags = eh.EH_INPUT_ON_DEVICE
    h = L.eh_load_edges_ex(ts.data_ptr(), td.data_ptr(), src.size, ctypes.byref(cfg))
    assert h
    try:
        assert L.eh_count_triangles(h) == ref
    finally:
        L.eh_free(h)


def test_release_cached_memory():
    import torch
    src, dst = synth.rmat(18, 16, 4400)
    eh.release_cached_memory()  # blocks cached by earlier tests
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info()[0]
    with eh.Graph(src, dst) as g:
        t = g.count_triangles()
    held = free0 - torch.cuda.mem_get_info()[0]
    assert held > 64 << 20  # the cache / pool keep the freed blocks
    eh.release_cached_memory()
    assert free0 - torch.cuda.mem_get_info()[0] < 8 << 20
    with eh.Graph(src, dst) as g:  # and the library still works afterwards
        assert g.count_triangles() == t


def test_triangles_per_vertex_out_checks():
    import torch
    src, dst = synth.rmat(10, 8, 4500)
    with eh.Graph(src, dst) as g:
        n = g.stats().n_active
        ref = g.triangles_per_vertex()
        with pytest.raises(TypeError):
            g.triangles_per_vertex(out=torch.zeros(n, dtype=torch.int32, device="cuda"))
        with pytest.raises(ValueError):
            g.triangles_per_vertex(out=torch.zeros(2 * n, dtype=torch.int64, device="cuda")[::2])
        with pytest.raises(TypeError):
            g.triangles_per_vertex(out=torch.zeros(n, dtype=torch.int64))
        out = torch.zeros(n, dtype=torch.int64, device="cuda")
        g.triangles_per_vertex(out=out)
        assert np.array_equal(out.cpu().numpy().astype(np.uint64), ref)


def test_count_batch_pipelined_uploads():
    """eh_count_batch: k lists (pinned and pageable host memory, empty and repeated
    lists), uploads overlapped with the work on the previous list; every count
    equals the oracle's."""
    import torch
    lists, ref = [], []
    for i, (sc, ef) in enumerate([(12, 16), (10, 8), (13, 16), (12, 16)]):
        src, dst = synth.rmat(sc, ef, 4600 + i)
        if i % 2 == 0:
            src = torch.from_numpy(src.view(np.int32)).pin_memory()
            dst = torch.from_numpy(dst.view(np.int32)).pin_memory()
        lists.append((src, dst))
        s_np = np.asarray(src).view(np.uint32) if not hasattr(src, "numpy") else src.numpy().view(np.uint32)
        d_np = np.asarray(dst).view(np.uint32) if not hasattr(dst, "numpy") else dst.numpy().view(np.uint32)
        ref.append((oracle.count_triangles(s_np, d_np), oracle.count_4cliques(s_np, d_np)))
    e = np.zeros(0, np.uint32)
    lists.insert(2, (e, e))
    ref.insert(2, (0, 0))
    lists.append(lists[0])
    ref.append(ref[0])
    assert eh.count_batch(lists) == [r[0] for r in ref]
    assert eh.count_batch(lists, "4cliques", stream=torch.cuda.Stream()) == [r[1] for r in ref]  # one lane
    assert eh.count_batch(lists, "4cliques") == [r[1] for r in ref]  # two lanes
    assert eh.count_batch([]) == []


def test_count_batch_lanes_with_different_sizes():
    """Two lanes loading graphs of different id widths at the same time launch the same
    ingest kernels with different dynamic shared-memory sizes; the per-kernel limit must
    never drop below what the other lane is about to launch with."""
    a, b = synth.rmat(8, 8, 4801), synth.rmat(13, 16, 4802)
    ra, rb = oracle.count_triangles(*a), oracle.count_triangles(*b)
    for _ in range(25):
        assert eh.count_batch([a, b, a, b, b, a]) == [ra, rb, ra, rb, rb, ra]


def test_count_batch_repeated_calls_release_lane_resources():
    """Every two-lane batch runs one lane on a fresh host thread whose side streams
    are destroyed at its exit: many calls in a row neither leak nor slow down."""
    src, dst = synth.rmat(10, 8, 4700)
    ref = oracle.count_triangles(src, dst)
    lists = [(src, dst)] * 3
    for _ in range(60):
        assert eh.count_batch(lists) == [ref] * 3
