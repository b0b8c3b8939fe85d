"""Small workload touching every kernel path, for compute-sanitizer (T7) and for
the bounds-checked build (EH_LIB=checked: lib/libeh_checked.so, csrc/check.cuh).

Checks counts against closed forms / the oracle so a sanitizer run is also a
parity run.  Usage: compute-sanitizer --tool memcheck python tools/sanitize_smoke.py
or EH_LIB=checked python tools/sanitize_smoke.py [--configs] (--configs adds the
C2-C4 loads and counts against the stored oracle values).
"""
import os
import sys
from math import comb

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import paper_1503_02368_b200 as eh  # noqa: E402
import synth  # noqa: E402


def check(src, dst, **kw):
    with eh.Graph(src, dst, **kw) as g:
        t, k = g.count_triangles(), g.count_4cliques()
        g.stats()
    og = oracle.Graph(src, dst)
    assert (t, k) == (og.count_triangles(), og.count_4cliques()), (t, k)
    og.close()
    return t, k


src, dst = synth.rmat(12, 16, 3)
check(src, dst)                                   # warp + CTA kernels, sort dedup
check(src, dst, tau=2)                            # mostly uint rows (STREAM / SEARCH)
check(src, dst, all_uint=True)
check(src, dst, bin_small_max=1, bin_large_min=1)  # everything in the CTA kernels
os.environ["EH_TEST_DEDUP"] = "hash"
check(src, dst)
del os.environ["EH_TEST_DEDUP"]
ids = np.random.default_rng(1).choice(2**32 - 1, size=2**13, replace=False).astype(np.uint32)
check(ids[src % ids.size], ids[dst % ids.size])   # dictionary path
s, d = synth.complete(1100)                       # |N+(x)| > 1024: K4 fallback kernel
with eh.Graph(s, d) as g:
    assert g.count_triangles() == comb(1100, 3)
    assert g.count_4cliques() == comb(1100, 4)
# NEXT rows, rank ranges, thread class, TMA-staged wide triangle kernels, the batch API
og = oracle.Graph(src, dst)
with eh.Graph(src, dst) as g:
    n = g.stats().n_active
    assert g.count_triangles_range(0, n // 2) == og.count_triangles_rank_range(0, n // 2)
    assert g.count_4cliques_range(n // 2, n) == og.count_4cliques_rank_range(n // 2, n)
    assert g.count_lollipop() == og.count_lollipop() and g.count_barbell() == og.count_barbell()
    assert g.count_triangles_unpruned() == og.count_triangles_unpruned()
    assert g.count_4cliques_unpruned() == og.count_4cliques_unpruned()
    g.alg_bytes_k4()
T = og.count_triangles()
with eh.Graph(src, dst, block_layout=True, order="bfs", bin_thread_max=16) as g:
    assert g.count_triangles() == T
os.environ["EH_TEST_TRI_WIDE"] = "1"
with eh.Graph(src, dst) as g:
    assert g.count_triangles() == T
ws, wd = synth.rmat(14, 16, 41)  # max |N+(x)| = 145: the wide shape's CTA classes
wT = oracle.count_triangles(ws, wd)
with eh.Graph(ws, wd) as g:
    assert g.count_triangles() == wT   # all of class 2 on the 4-warp (mid) CTAs
    os.environ["EH_TEST_TRI_MID"] = "135"  # mid and big (16-warp, TMA-staged) CTA classes both populated
    assert g.count_triangles() == wT
    os.environ["EH_TEST_TRI_MID"] = "0"  # all of class 2 on the 16-warp CTAs
    assert g.count_triangles() == wT
    del os.environ["EH_TEST_TRI_MID"]
del os.environ["EH_TEST_TRI_WIDE"]
assert eh.count_batch([(src, dst), (src[:1000], dst[:1000]), (src, dst)])[0] == T
og.close()
e = np.zeros(0, np.uint32)
with eh.Graph(e, e) as g:
    assert g.count_triangles() == 0 and g.count_4cliques() == 0
rng = np.random.default_rng(2)
for t in range(200):
    a = np.unique(rng.integers(0, int(rng.choice([100, 10**5, 2**32])), int(rng.integers(0, 3000)), dtype=np.uint64))
    b = np.unique(rng.integers(0, int(rng.choice([100, 10**5, 2**32])), int(rng.integers(0, 3000)), dtype=np.uint64))
    a = a.astype(np.uint32)
    b = b.astype(np.uint32)
    assert np.array_equal(eh.intersect(a, b), np.intersect1d(a, b))
if "--configs" in sys.argv:
    import json
    gold = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests",
                                       "golden", "configs_oracle.json")))["configs"]
    for name in ("C2", "C3", "C4"):
        cs, cd = synth.CONFIGS[name].generate()
        with eh.Graph(cs, cd) as g:
            assert g.count_triangles() == gold[name]["triangles"], name
            assert g.count_4cliques() == gold[name]["four_cliques"], name
            n = g.stats().n_active
            assert g.count_4cliques_range(0, n // 2) + g.count_4cliques_range(n // 2, n) == gold[name]["four_cliques"]
        print(name, "ok", flush=True)
print("sanitize smoke ok", eh.eh.LIB_PATH)
