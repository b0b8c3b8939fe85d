"""Write tests/golden/rank_ranges_oracle.json: the CPU ORACLE's triangle and
4-clique counts over sampled RANK RANGES of a config (eh_oracle.c "Rank
ranges": the cliques whose earliest vertex, in the ascending (degree, original
id) order, has a rank in [r0, r1)).

Where the full oracle 4-clique count is out of reach (C5: 1.31 B edges; the
full nest would take days on this host), these are the sampled outputs the
CUDA path's eh_count_*_range are checked against, on the full graph in the
launch configuration bench.py times.  Calls only synth/ (inputs) and oracle/
(counts, ranks, out-degrees) -- never the CUDA path.  Windows: the lowest ranks,
windows at 1/4, 1/2, 3/4 and 9/10 of the rank space, the ranks around the
largest out-degree, the 16 single ranks of largest out-degree (the hub-row
path of the 4-clique kernels when |N+(x)| > 1024), and the highest ranks.
Usage:  python tools/write_oracle_rank_goldens.py C5 [C3 ...]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import synth  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "rank_ranges_oracle.json")


BUDGET = 4e11  # per window: sum of |N+(x)|^3 (a bound on the K4 nest's work; C2 measured ~5e9 per s on 8 threads)


def windows(dplus: np.ndarray):
    """Rank windows, each shrunk until its cost proxy sum |N+(x)|^3 fits BUDGET."""
    n = dplus.size
    c3 = np.concatenate([[0.0], np.cumsum(dplus.astype(np.float64) ** 3)])

    def fwd(a, b):  # [a, b') with b' <= b as large as the budget allows (>= 1 rank)
        b2 = int(np.searchsorted(c3, c3[a] + BUDGET, side="right")) - 1
        return a, max(a + 1, min(b, b2))

    def bwd(a, b):  # [a', b) with a' >= a
        a2 = int(np.searchsorted(c3, c3[b] - BUDGET, side="left"))
        return min(b - 1, max(a, a2)), b

    w = [fwd(0, min(n, 1 << 16))]
    for f in (0.25, 0.5, 0.75, 0.9):
        a = int(n * f)
        w.append(fwd(a, min(n, a + (1 << 14))))
    rmax = int(np.argmax(dplus))
    w.append(fwd(max(0, rmax - 4), min(n, rmax + 4)))
    for r in np.argsort(dplus, kind="stable")[::-1][:16].tolist():
        w.append((int(r), int(r) + 1))
    w.append(bwd(max(0, n - 4096), n))
    return w


def main(names):
    data = json.load(open(OUT)) if os.path.exists(OUT) else {
        "citation": "eh_oracle.c 'Rank ranges' (loop nests PAPER.md:538-542 and PAPER.md:217 with the earliest "
                    "vertex x restricted to a rank window of the (degree, original id) order, SURVEY.md §8(c) "
                    "step 3); written by tools/write_oracle_rank_goldens.py from synth/ + oracle/ only",
        "configs": {}}
    for name in names:
        cfg = synth.CONFIGS[name]
        t0 = time.time()
        src, dst = cfg.generate()
        ck = synth.checksum(src, dst)
        g = oracle.Graph(src, dst)
        del src, dst
        t1 = time.time()
        print(f"{name}: oracle ingest {t1 - t0:.0f} s", flush=True)
        vid, _, off, _ = g.export(with_adj=False)
        ids = g.rank_ids()
        idx = np.searchsorted(vid, ids)
        dplus = (off[idx + 1] - off[idx]).astype(np.int64)
        del vid, off, ids, idx
        entry = {"checksum": str(ck), "n_active": g.n_vertices, "ingest_seconds": round(t1 - t0, 1),
                 "windows": []}
        for r0, r1 in windows(dplus):
            ts = time.time()
            tri = g.count_triangles_rank_range(r0, r1)
            k4 = g.count_4cliques_rank_range(r0, r1)
            rec = {"r0": r0, "r1": r1, "max_out_degree": int(dplus[r0:r1].max()), "triangles": tri,
                   "four_cliques": k4, "seconds": round(time.time() - ts, 1)}
            entry["windows"].append(rec)
            print(name, rec, flush=True)
            data["configs"][name] = entry
            json.dump(data, open(OUT, "w"), indent=1)
        g.close()


if __name__ == "__main__":
    main(sys.argv[1:] or ["C5"])
