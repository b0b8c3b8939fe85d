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
names = sys.argv[1:] or ["C1", "C2", "C3", "C4", "C5"]
reps = 5
for name in names:
    cfg = synth.CONFIGS[name]
    src, dst = cfg.generate()
    n_in = src.size
    s = torch.from_numpy(src.view(np.int32)).cuda()
    d = torch.from_numpy(dst.view(np.int32)).cuda()
    del src, dst
    st = torch.cuda.Stream()
    loads, tris, k4s = [], [], []
    res = {}
    for r in range(reps + 1):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        with torch.cuda.stream(st):
            e[0].record(st)
            g = eh.Graph(s, d, stream=st)
            e[1].record(st)
            t = g.count_triangles()
            e[2].record(st)
            k = g.count_4cliques() if cfg.query == "4cliques" else None
            e[3].record(st)
            st.synchronize()
            if r == 0:
                stats = g.stats()
            g.close()
        if r == 0:
            res.update(triangles=t, four_cliques=k)
            continue
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
    print(json.dumps(res), flush=True)
    del s, d
    torch.cuda.empty_cache()
