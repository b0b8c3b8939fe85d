"""Dev aid: time eh_triangles_per_vertex on one config under EH_PV_AND / EH_PV_ANDW settings."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1503_02368_b200 as eh  # noqa: E402
import synth  # noqa: E402

if os.environ.get("TRI_LIB"):  # dev: time another build of the library
    import paper_1503_02368_b200.eh as _ehm
    _ehm.LIB_PATH = os.environ["TRI_LIB"]

name = sys.argv[1]
settings = sys.argv[2:]
src, dst = synth.CONFIGS[name].generate()
s = torch.from_numpy(src.view(np.int32)).cuda()
d = torch.from_numpy(dst.view(np.int32)).cuda()
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    g = eh.Graph(s, d, stream=st)
    tv = torch.empty(g.stats().n_active, dtype=torch.int64, device="cuda")
    ref = None
    for sett in settings:
        a, w, m = (sett.split(",") + ["0"])[:3]
        os.environ["EH_PV_AND"], os.environ["EH_PV_ANDW"], os.environ["EH_PV_MODE"] = a, w, m
        ts = []
        for r in range(6):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            g.triangles_per_vertex(tv)
            e1.record(st)
            st.synchronize()
            if r:
                ts.append(e0.elapsed_time(e1))
        h = int(tv.sum())
        ref = ref or h
        if m != "0":
            ref = None
        print(name, sett, f"{statistics.median(ts):.3f} ms", "ok" if h == ref else "MISMATCH", flush=True)
