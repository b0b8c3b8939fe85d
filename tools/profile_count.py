"""Profiling driver (development aid): load one config, then call the count
entry point `--reps` times.  Run under ncu with -k regex:k_tri / k_k4."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import synth  # noqa: E402
import paper_1503_02368_b200 as eh  # noqa: E402

if os.environ.get("TRI_LIB"):  # dev: profile another build of the library
    import paper_1503_02368_b200.eh as _ehm
    _ehm.LIB_PATH = os.environ["TRI_LIB"]

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--query", default="tri", choices=["tri", "k4", "pv", "lollipop", "unpruned"])
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--tau", type=int, default=0)
ap.add_argument("--small", type=int, default=0)
ap.add_argument("--large", type=int, default=0)
ap.add_argument("--small_max", type=int, default=0)
a = ap.parse_args()
src, dst = synth.CONFIGS[a.config].generate()
with eh.Graph(src, dst, tau=a.tau, bin_small_max=a.small or a.small_max, bin_large_min=a.large) as g:
    st = g.stats()
    for _ in range(a.reps):
        t0 = time.perf_counter()
        c = {"tri": g.count_triangles, "k4": g.count_4cliques, "lollipop": g.count_lollipop,
             "pv": lambda: int(g.triangles_per_vertex().sum()),
             "unpruned": g.count_triangles_unpruned}[a.query]()
        print(f"{a.query} = {c}  {1e3 * (time.perf_counter() - t0):.2f} ms", flush=True)
    print(st, flush=True)
