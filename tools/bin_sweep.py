"""Dev aid: eh_count_triangles time vs the warp/CTA class boundary (bin_large_min)."""
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
src, dst = synth.CONFIGS[name].generate()
s = torch.from_numpy(src.view(np.int32)).cuda()
d = torch.from_numpy(dst.view(np.int32)).cuda()
st = torch.cuda.Stream()
what = os.environ.get("WHAT", "tri")
for lm in sys.argv[2:]:
    with torch.cuda.stream(st):
        g = eh.Graph(s, d, stream=st, **{os.environ.get("KNOB", "bin_large_min"): int(lm)})
        f = {"tri": g.count_triangles, "k4": g.count_4cliques, "pv": lambda: int(g.triangles_per_vertex().sum())}[what]
        ts = []
        for r in range(6):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            c = f()
            e1.record(st)
            st.synchronize()
            if r:
                ts.append(e0.elapsed_time(e1))
        g.close()
    print(name, what, os.environ.get("KNOB", "bin_large_min"), lm, f"{statistics.median(ts):.3f} ms", c, flush=True)
