"""Intersection microbenchmarks in the shape of the paper's layout / algorithm studies,
run through the REAL count kernels (dev aid; results in profiles/, discussed in DESIGN.md):

  E2   uint vs bitset intersection time vs density (Fig. `fig:impact_density`,
       PAPER.md:611-618): |A| = 960, |B| = 2048, range R swept (|A| = 960 keeps
       N+(x) = A ++ 32 row ends within the 1024 elements the 4-warp CTA's 8 KB table
       can hash at load 1/2 -- every C1-C4 set is; above it the kernel falls back to a
       binary search of the staged list, which "--cardA 2048" shows);
  E16a uint algorithms vs cardinality ratio (Fig. `fig:card_skew2`):
       range 1M, |A| = 64, |B| swept;
  E16b uint algorithms vs density at fixed cardinality (PAPER.md:1603-1608,
       Fig. `fig:uint_fixedcard2`): |A| = 960, |B| = 2048, range 10K - 1.2M.

A single pair of such sets is launch-bound on a GPU, so each point is a BATCH of rows
|A(x) cap B(y)| laid out as a graph and counted by eh_count_triangles: ids X < Y < Z,
edges (x, y) for the rows, (x, z) for z in A(x), (y, z) for z in B(y), loaded with
order="id" (EH_ORDER_ID: edges point low -> high id), so N+(x) = Y(x) ++ A(x),
N+(y) = B(y), N+(z) = {} and T = sum over rows of |A(x) cap B(y)| (the later y' of x ride
along in A: at most `rows_per_x` - 1 extra probes per row).  Modes = the library's own
layout / algorithm switches: uint auto (EH_ALL_UINT), stream only (EH_NO_ALGO, "-RA"),
search only (EH_FORCE_SEARCH), bitset (tau = 2^20), default (tau = 128).  The count is
checked against numpy on the first point of each sweep and across modes everywhere.

  python tools/intersect_bench.py [E2|E16a|E16b ...] > profiles/r2_intersect_micro.jsonl
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1503_02368_b200 as eh  # noqa: E402

MODES = {
    "uint_auto": dict(all_uint=True),
    "uint_stream": dict(no_algo=True),
    "uint_search": dict(force_search=True),
    "bitset": dict(tau=1 << 20),
    "default_tau128": dict(),
}


def sample_sets(rng, nsets, card, R):
    """nsets sorted sets of `card` distinct values in [0, R) (numpy Generator.choice)."""
    out = np.empty((nsets, card), np.uint32)
    for i in range(nsets):
        out[i] = np.sort(rng.choice(R, card, replace=False))
    return out


def build(nx, ny, rows_per_x, cardA, cardB, R, seed):
    rng = np.random.default_rng(seed)
    A = sample_sets(rng, nx, cardA, R)
    B = sample_sets(rng, ny, cardB, R)
    ys = np.empty((nx, rows_per_x), np.uint32)
    for i in range(nx):
        ys[i] = rng.choice(ny, rows_per_x, replace=False)
    x0, y0, z0 = 0, nx, nx + ny
    xs = np.arange(nx, dtype=np.uint32)
    src = np.concatenate([np.repeat(xs, rows_per_x), np.repeat(xs, cardA),
                          np.repeat(np.arange(ny, dtype=np.uint32) + y0, cardB)])
    dst = np.concatenate([(ys + y0).ravel(), (A + z0).ravel(), (B + z0).ravel()])
    return src.astype(np.uint32), dst.astype(np.uint32), A, B, ys


def numpy_count(A, B, ys, limit=20000):
    if ys.size > limit:
        return None
    t = 0
    for x in range(ys.shape[0]):
        for y in ys[x]:
            t += np.intersect1d(A[x], B[y], assume_unique=True).size
    return t


def time_modes(src, dst, reps=5):
    s = torch.from_numpy(src.view(np.int32)).cuda()
    d = torch.from_numpy(dst.view(np.int32)).cuda()
    res, counts = {}, {}
    for name, kw in MODES.items():
        with eh.Graph(s, d, order="id", **kw) as g:
            c = g.count_triangles()  # warm-up
            ts = []
            for _ in range(reps):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                c2 = g.count_triangles()
                ts.append((time.perf_counter() - t0) * 1e3)
            assert c2 == c
            st = g.stats()
        counts[name] = c
        res[name] = min(ts)
    assert len(set(counts.values())) == 1, counts
    return res, counts["uint_auto"], st


def point(exp, nx, ny, k, cardA, cardB, R, seed, check):
    src, dst, A, B, ys = build(nx, ny, k, cardA, cardB, R, seed)
    ms, count, st = time_modes(src, dst)
    if check:
        ref = numpy_count(A, B, ys)
        assert ref is None or ref == count, (ref, count)
    rows = nx * k
    rec = {"exp": exp, "cardA": cardA, "cardB": cardB, "range": R, "density": round(cardB / R, 6), "rows": rows,
           "n_active": int(st.n_active), "hits": int(count), "checked_vs_numpy": bool(check and ys.size <= 20000)}
    for name, t in ms.items():
        rec[name + "_ms"] = round(t, 4)
        rec[name + "_ns_per_row"] = round(t * 1e6 / rows, 2)
    print(json.dumps(rec), flush=True)


def main():
    args = sys.argv[1:]
    cardA = 960
    if "--cardA" in args:
        i = args.index("--cardA")
        cardA = int(args[i + 1])
        del args[i:i + 2]
    exps = args or ["E2", "E16a", "E16b"]
    if "E2" in exps or "E16b" in exps:
        # |B| = 2048; E2 sweeps the dense end, E16b the paper's 10K - 1.2M
        ranges = {"E2": [2560, 4096, 8192, 16384, 32768, 65536, 131072, 262144, 524288],
                  "E16b": [10000, 20000, 50000, 100000, 200000, 400000, 800000, 1200000]}
        for exp in ("E2", "E16b"):
            if exp not in exps:
                continue
            point(exp + "-check", 512, 512, 32, cardA, 2048, ranges[exp][0], 99, True)
            for i, R in enumerate(ranges[exp]):
                point(exp, 4096, 4096, 32, cardA, 2048, R, 100 + i, False)
    if "E16a" in exps:
        point("E16a-check", 2048, 4096, 8, 64, 64, 1 << 20, 199, True)
        for i, cb in enumerate([64, 128, 256, 384, 512, 768, 1024, 2048, 4096, 16384, 65536, 262144]):
            ny = max(16, min(4096, (1 << 24) // cb))
            point("E16a", 65536, ny, 8, 64, cb, 1 << 20, 200 + i, False)


if __name__ == "__main__":
    main()
