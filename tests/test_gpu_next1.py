"""GPU parity for SURVEY.md §8(f) NEXT-1: per-vertex triangle counts t(v) and the
Lollipop L3,1 / Barbell B3,1 COUNT(*), CUDA path
through the C ABI vs the oracle, bit-exact (integers).

The GPU reports t(v) per rank; export()'s orig_id maps ranks to original ids and
the oracle reports t(v) per sorted original id, so the comparison is by id.
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


def _gpu(src, dst, **kw):
    with eh.Graph(src, dst, **kw) as g:
        t = g.triangles_per_vertex()
        orig = g.export()[2]
        order = np.argsort(orig, kind="stable")
        return orig[order], t[order], g.count_lollipop(), g.count_barbell(), g.count_triangles()


def _check(src, dst, **kw):
    ids, t, lol, bar, tri = _gpu(src, dst, **kw)
    og = oracle.Graph(src, dst)
    try:
        vid, _, _, _ = og.export()
        assert np.array_equal(ids, vid)
        ot = og.triangles_per_vertex()
        assert np.array_equal(t, ot), np.flatnonzero(t != ot)[:10]
        assert int(t.sum()) == 3 * tri  # every triangle credited to its three vertices
        assert lol == og.count_lollipop()
        assert bar == og.count_barbell()
    finally:
        og.close()
    return t, lol, bar


@pytest.mark.parametrize("n", list(range(0, 20)) + [33, 64, 129, 300])
def test_kn_closed_forms(n):
    ids, t, lol, bar, _ = _gpu(*synth.complete(n))
    tv = comb(n - 1, 2) if n else 0
    assert ids.size == (n if n >= 2 else 0)
    assert np.all(t == tv)
    assert lol == n * 2 * tv * (n - 1)
    assert bar == n * (n - 1) * (2 * tv) ** 2


def test_k1700_barbell_above_2_64():
    n = 1700
    _, t, lol, bar, _ = _gpu(*synth.complete(n))
    tv = comb(n - 1, 2)
    assert np.all(t == tv)
    assert bar == n * (n - 1) * (2 * tv) ** 2 > 2**64
    assert lol == n * 2 * tv * (n - 1)


def test_multipartite_degree_above_stage_cap():
    # K_{a,a,a}: all degrees 2a, so |N+(x)| runs up to 2a - 1 = 4199, above the CTA kernel's
    # default staging capacity (2048; it grows to the next power of two); t(v) = a^2.
    a = 2100
    _, t, lol, bar, tri = _gpu(*synth.complete_multipartite((a, a, a)))
    assert tri == a**3 and np.all(t == a * a)
    assert lol == 3 * a * 2 * a * a * (2 * a)
    assert bar == 3 * a * (2 * a) * (2 * a * a) ** 2


def test_multipartite_small_vs_oracle():
    for sizes in [(3, 4), (5, 5, 5), (2, 3, 4, 5), (30, 40, 50), (7, 1, 3, 2, 6, 9)]:
        _check(*synth.complete_multipartite(sizes))


@pytest.mark.parametrize("seed", range(20))
def test_random_er(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(2, 600))
    p = float(rng.choice([0.002, 0.01, 0.05, 0.2]))
    _check(*synth.er(n, p, seed))


@pytest.mark.parametrize("scale,ef,seed", [(s, ef, seed) for s in (6, 10, 14, 16) for ef in (4, 16)
                                           for seed in range(2)])
def test_random_rmat(scale, ef, seed):
    _check(*synth.rmat(scale, ef, 1000 * scale + 10 * ef + seed))


@pytest.mark.parametrize("seed", range(6))
def test_random_multigraph_with_noise(seed):
    src, dst = synth.random_graph(int(np.random.default_rng(seed).integers(3, 3000)), 20000, seed)
    _check(src, dst)


def test_empty_and_degenerate():
    e = np.zeros(0, np.uint32)
    ids, t, lol, bar, _ = _gpu(e, e)
    assert ids.size == 0 and t.size == 0 and lol == 0 and bar == 0
    loops = np.arange(50, dtype=np.uint32)
    assert _gpu(loops, loops)[2:4] == (0, 0)
    tri = (np.array([0, 1, 2], np.uint32), np.array([1, 2, 0], np.uint32))
    ids, t, lol, bar, _ = _gpu(*tri)
    assert list(t) == [1, 1, 1] and lol == 3 * 2 * 2 and bar == 6 * 4  # K3: B = n(n-1)(2t)^2
    # triangle plus a pendant edge at vertex 0
    _check(np.array([0, 1, 2, 0], np.uint32), np.array([1, 2, 0, 7], np.uint32))


def test_star_with_path_hub():
    s, d = synth.star(100_000)
    leaves = np.arange(1, 100_001, dtype=np.uint32)
    s = np.concatenate([s, leaves[:-1]])
    d = np.concatenate([d, leaves[1:]])
    _check(s, d)


@pytest.mark.parametrize("kw", [dict(tau=256), dict(tau=2), dict(tau=1 << 20), dict(all_uint=True), dict(no_algo=True), dict(force_search=True),
                                dict(bin_small_max=2**32 - 1), dict(bin_large_min=1), dict(min_bitset_card=1)])
def test_layout_and_binning_invariance(kw):
    src, dst = synth.rmat(13, 16, 4242)
    base = _gpu(src, dst)
    other = _gpu(src, dst, **kw)
    assert np.array_equal(base[1], other[1]) and base[2:] == other[2:]


def test_device_output_tensor():
    torch = pytest.importorskip("torch")
    src, dst = synth.rmat(12, 8, 99)
    with eh.Graph(src, dst) as g:
        host = g.triangles_per_vertex()
        out = torch.full((host.size + 5,), -1, dtype=torch.int64, device="cuda")
        dev = g.triangles_per_vertex(out)
        assert np.array_equal(dev.cpu().numpy().astype(np.uint64), host)
        assert int(out[host.size:].eq(-1).sum()) == 5  # nothing written past n_active


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_config_vs_oracle(name, golden_dir):
    gold = json.load(open(os.path.join(golden_dir, "configs_oracle.json")))["configs"][name]
    src, dst = synth.CONFIGS[name].generate()
    assert str(synth.checksum(src, dst)) == gold["checksum"]
    t, _, _ = _check(src, dst)
    assert int(t.sum()) == 3 * gold["triangles"]


@pytest.mark.parametrize("seed", range(2))
def test_unstaged_cta_path(seed, monkeypatch):
    # EH_TEST_PV_XCAP (test hook) lowers the CTA kernel's staging capacity, so every
    # |N+(x)| > 128 takes the unstaged path (global N+(x), global credit atomics).
    monkeypatch.setenv("EH_TEST_PV_XCAP", "128")
    _check(*synth.rmat(14, 16, 777 + seed))
    a = 300
    _, t, lol, bar, tri = _gpu(*synth.complete_multipartite((a, a, a)))
    assert tri == a**3 and np.all(t == a * a)


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4"])
def test_config_vs_oracle_next1_golden(name, golden_dir):
    """Full-size configs against the oracle's stored NEXT-1 values
    (tools/write_oracle_goldens.py --next1): Lollipop, Barbell and the sha256 of
    t(v) in ascending original-id order."""
    import hashlib
    gold = json.load(open(os.path.join(golden_dir, "configs_oracle.json")))["configs"].get(name, {})
    if "next1" not in gold:
        pytest.skip(f"no stored NEXT-1 oracle values for {name}")
    src, dst = synth.CONFIGS[name].generate()
    assert str(synth.checksum(src, dst)) == gold["checksum"]
    ids, t, lol, bar, tri = _gpu(src, dst)
    assert tri == gold["triangles"]
    assert int(t.sum()) == gold["next1"]["sum_t"] == 3 * tri
    assert hashlib.sha256(t.astype("<u8").tobytes()).hexdigest() == gold["next1"]["t_sha256"]
    assert lol == int(gold["next1"]["lollipop"]) and bar == int(gold["next1"]["barbell"])
