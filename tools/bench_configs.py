"""Per-config measurements (development/evidence, not the driver's bench):
for each BASELINE config, device-resident inputs, CUDA-event times of
eh_load_edges and of the count(s), B_tri and the roofline fraction.
Writes one JSON object per config to stdout."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1503_02368_b200 as eh  # noqa: E402
import synth  # noqa: E402

PEAK = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")) else 6538.6
NEXT1 = "--next1" in sys.argv
NEXT2 = "--next2" in sys.argv
NEXT3 = "--next3" in sys.argv
NEXT4 = "--next4" in sys.argv
K4ALL = "--k4" in sys.argv  # 4-clique count (and B_K4) on every config, not only C4
names = [a for a in sys.argv[1:] if not a.startswith("--")] or ["C1", "C2", "C3", "C4", "C5"]
reps = 5
for name in names:
    cfg = synth.CONFIGS[name]
    k4_reps = 1 if name == "C5" else reps  # C5's 4-clique count: one timed run
    src, dst = cfg.generate()
    n_in = src.size
    s = torch.from_numpy(src.view(np.int32)).cuda()
    d = torch.from_numpy(dst.view(np.int32)).cuda()
    del src, dst
    st = torch.cuda.Stream()
    loads, tris, k4s, pvs, lols, bars = [], [], [], [], [], []
    res = {}
    for r in range(reps + 1):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        with torch.cuda.stream(st):
            e[0].record(st)
            g = eh.Graph(s, d, stream=st)
            e[1].record(st)
            t = g.count_triangles()
            e[2].record(st)
            k = g.count_4cliques() if (cfg.query == "4cliques" or K4ALL) and (r <= k4_reps) else None
            e[3].record(st)
            if NEXT1:  # t(v) into a device array, Lollipop, Barbell
                e += [torch.cuda.Event(enable_timing=True) for _ in range(4)]
                tv = torch.empty(g.stats().n_active if r == 0 else tv.numel(), dtype=torch.int64, device="cuda")
                e[4].record(st)
                g.triangles_per_vertex(tv)
                e[5].record(st)
                lol = g.count_lollipop()
                e[6].record(st)
                bar = g.count_barbell()
                e[7].record(st)
            st.synchronize()
            if r == 0:
                stats = g.stats()
                if k is not None and stats.n_active <= (1 << 24):
                    b_k4 = g.alg_bytes_k4()
            g.close()
        if r == 0:
            res.update(triangles=t, four_cliques=k)
            if NEXT1:
                res.update(lollipop=str(lol), barbell=str(bar), sum_t=int(tv.sum()))
            continue
        if NEXT1:
            pvs.append(e[4].elapsed_time(e[5]))
            lols.append(e[5].elapsed_time(e[6]))
            bars.append(e[6].elapsed_time(e[7]))
        loads.append(e[0].elapsed_time(e[1]))
        tris.append(e[1].elapsed_time(e[2]))
        if k is not None:
            k4s.append(e[2].elapsed_time(e[3]))
    lt, tt = statistics.median(loads), statistics.median(tris)
    res.update(config=name, n_input=int(n_in), m=stats.m_undirected, n_active=stats.n_active,
               max_out_degree=stats.max_out_degree, load_ms=lt, tri_ms=tt,
               alg_bytes_tri=stats.alg_bytes_tri, tri_gbs=stats.alg_bytes_tri / tt / 1e6,
               tri_roofline_frac=stats.alg_bytes_tri / tt / 1e6 / PEAK,
               step_edges_per_s=n_in / ((lt + tt) / 1e3), count_edges_per_s=n_in / (tt / 1e3))
    if k4s:
        res["k4_ms"] = statistics.median(k4s)
        if stats.n_active <= (1 << 24):
            res.update(alg_bytes_k4=b_k4, k4_gbs=b_k4 / res["k4_ms"] / 1e6,
                       k4_roofline_frac=b_k4 / res["k4_ms"] / 1e6 / PEAK)
    if pvs:
        pv = statistics.median(pvs)
        pv_bytes = stats.alg_bytes_tri + 8 * stats.n_active  # B_tri reads + the t(v) array
        res.update(pv_ms=pv, lollipop_ms=statistics.median(lols), barbell_ms=statistics.median(bars),
                   pv_alg_bytes=pv_bytes, pv_gbs=pv_bytes / pv / 1e6, pv_roofline_frac=pv_bytes / pv / 1e6 / PEAK)
    if NEXT2:  # unpruned nest on the symmetric trie, default and all-uint (-R)
        for label, kw in (("", {}), ("_R", {"all_uint": True})):
            with torch.cuda.stream(st):
                g = eh.Graph(s, d, stream=st, **kw)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                sst = g.symmetric_stats()  # builds the symmetric trie (+ its statistics)
                e1.record(st)
                st.synchronize()
                build_ms = e0.elapsed_time(e1)
                u = g.count_triangles_unpruned()
                us, ps = [], []
                for r in range(reps):
                    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
                    ev[0].record(st)
                    g.count_triangles_unpruned()
                    ev[1].record(st)
                    g.count_triangles()
                    ev[2].record(st)
                    st.synchronize()
                    us.append(ev[0].elapsed_time(ev[1]))
                    ps.append(ev[1].elapsed_time(ev[2]))
                g.close()
            um = statistics.median(us)
            if label == "" and (cfg.query == "4cliques" or name in ("C1", "C2")):
                with torch.cuda.stream(st):
                    g = eh.Graph(s, d, stream=st)
                    g.symmetric_stats()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(st)
                    res["k4_unpruned"] = g.count_4cliques_unpruned()
                    e1.record(st)
                    st.synchronize()
                    res["k4_unpruned_ms"] = e0.elapsed_time(e1)
                    g.close()
            res.update({f"unpruned{label}": u, f"unpruned{label}_ms": um, f"pruned{label}_ms": statistics.median(ps),
                        f"sym_build{label}_ms": build_ms, f"B_sym{label}": sst.alg_bytes_tri,
                        f"unpruned{label}_gbs": sst.alg_bytes_tri / um / 1e6,
                        f"unpruned{label}_frac": sst.alg_bytes_tri / um / 1e6 / PEAK,
                        f"sym_bitset_sets{label}": sst.n_bitset_sets, f"sym_max_degree": sst.max_out_degree})
    if NEXT3:  # relation / set / block level layouts, -R and -RA ablations
        for label, kw in (("set", {}), ("R", {"all_uint": True}), ("RA", {"no_algo": True}),
                          ("block", {"block_layout": True})):
            with torch.cuda.stream(st):
                ts, lt, ks, ls = [], [], [], []
                for r in range(reps):
                    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
                    ev[0].record(st)
                    g = eh.Graph(s, d, stream=st, **kw)
                    ev[1].record(st)
                    tv = g.count_triangles()
                    ev[2].record(st)
                    kv = g.count_4cliques() if cfg.query == "4cliques" and label != "block" else None
                    ev[3].record(st)
                    lv = g.count_lollipop() if label != "block" else None
                    ev[4].record(st)
                    st.synchronize()
                    g.close()
                    lt.append(ev[0].elapsed_time(ev[1]))
                    ts.append(ev[1].elapsed_time(ev[2]))
                    ks.append(ev[2].elapsed_time(ev[3]))
                    ls.append(ev[3].elapsed_time(ev[4]))
                assert tv == res["triangles"], (label, tv)
                res[f"layout_{label}"] = {"load_ms": statistics.median(lt), "tri_ms": statistics.median(ts),
                                          "k4_ms": statistics.median(ks) if kv is not None else None,
                                          "k4": kv, "lollipop_ms": statistics.median(ls) if lv is not None else None,
                                          "lollipop": str(lv) if lv is not None else None}
    if NEXT4:  # node orderings
        for order in ("degree", "random", "bfs", "hybrid", "shingle", "rev_degree"):
            row = {}
            for label, kw in (("", {}), ("_R", {"all_uint": True})):
                with torch.cuda.stream(st):
                    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
                    ev[0].record(st)
                    g = eh.Graph(s, d, stream=st, order=order, **kw)
                    ev[1].record(st)
                    tv = g.count_triangles()
                    ev[2].record(st)
                    uv = g.count_triangles_unpruned() if name != "C5" else None
                    ev[3].record(st)
                    st.synchronize()
                    mo = g.stats().max_out_degree
                    g.close()
                assert tv == res["triangles"] and (uv is None or uv == 6 * tv), (order, tv, uv)
                row.update({f"load{label}_ms": ev[0].elapsed_time(ev[1]), f"pruned{label}_ms": ev[1].elapsed_time(ev[2]),
                            f"unpruned{label}_ms": ev[2].elapsed_time(ev[3]) if uv is not None else None,
                            "max_out_degree": mo})
            res[f"order_{order}"] = row
    print(json.dumps(res), flush=True)
    del s, d
    torch.cuda.empty_cache()
