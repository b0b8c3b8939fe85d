"""The CPU oracle timed by the paper's protocol (each time is the
mean of 7 runs after dropping the fastest and slowest; loading / index creation
excluded and reported separately) on this host -- the reported CPU baseline of
SURVEY.md §8(d) "Oracle timing beside it": all host threads for C1-C4 (4-cliques
on C4, 3 runs), plus a single-threaded count for C1-C3 (one run at C3), with the
host's core count and CPU model.  One JSON object per line on stdout.
Calls only synth/ and oracle/.  Usage: python tools/oracle_protocol.py [C1 C2 ...]
"""
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import synth  # noqa: E402


def cpu_model():
    for ln in open("/proc/cpuinfo"):
        if ln.startswith("model name"):
            return ln.split(":", 1)[1].strip()
    return "unknown"


def timed(f, runs):
    ts, vals = [], set()
    for _ in range(runs):
        t0 = time.perf_counter()
        vals.add(f())
        ts.append(time.perf_counter() - t0)
    kept = sorted(ts)[1:-1] if runs >= 3 else ts
    assert len(vals) == 1, vals
    return vals.pop(), statistics.mean(kept), ts


def main(names):
    threads = oracle.default_threads()
    for name in names:
        cfg = synth.CONFIGS[name]
        src, dst = cfg.generate()
        n_in = int(src.size)
        t0 = time.perf_counter()
        g = oracle.Graph(src, dst)
        t_ing = time.perf_counter() - t0
        rec = {"config": name, "n_input": n_in, "host_threads": threads, "cpu": cpu_model(),
               "ingest_s": t_ing, "ingest_threads": 1}
        t, m, ts = timed(lambda: g.count_triangles(threads), 7)
        rec.update(triangles=t, tri_s=m, tri_runs_s=ts, tri_edges_per_s=n_in / m)
        if name in ("C1", "C2", "C3"):
            runs = 1 if name == "C3" else 3
            _, m1, ts1 = timed(lambda: g.count_triangles(1), runs)
            rec.update(tri_1thread_s=m1, tri_1thread_runs_s=ts1)
        if cfg.query == "4cliques":
            k, mk, tk = timed(lambda: g.count_4cliques(threads), 3)
            rec.update(four_cliques=k, k4_s=mk, k4_runs_s=tk, k4_edges_per_s=n_in / mk)
        g.close()
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["C1", "C2", "C3", "C4"])
