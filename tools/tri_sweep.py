"""Dev aid: time eh_count_triangles (TRI_QUERY=k4: eh_count_4cliques) on one config under several
values of an environment switch ("-" = unset); TRI_LIB=path times another build of the library."""
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

name, var = sys.argv[1], sys.argv[2]
src, dst = synth.CONFIGS[name].generate()
s = torch.from_numpy(src.view(np.int32)).cuda()
d = torch.from_numpy(dst.view(np.int32)).cuda()
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    g = eh.Graph(s, d, stream=st)
    ref = None
    for val in sys.argv[3:]:
        if val == "-":
            os.environ.pop(var, None)  # "-": the variable unset
        else:
            os.environ[var] = val
        ts = []
        for r in range(6):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            c = g.count_4cliques() if os.environ.get("TRI_QUERY") == "k4" else g.count_triangles()
            e1.record(st)
            st.synchronize()
            if r:
                ts.append(e0.elapsed_time(e1))
        ref = ref or c
        print(name, var, val, f"{statistics.median(ts):.3f} ms", "ok" if c == ref else "MISMATCH", flush=True)
