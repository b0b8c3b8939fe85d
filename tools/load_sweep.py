"""Dev aid: eh_load_edges time (device-resident inputs, CUDA events) on one config
under several values of an environment switch ("-" = unset)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1503_02368_b200 as eh  # noqa: E402
import synth  # noqa: E402

name, var = sys.argv[1], sys.argv[2]
src, dst = synth.CONFIGS[name].generate()
s = torch.from_numpy(src.view(np.int32)).cuda()
d = torch.from_numpy(dst.view(np.int32)).cuda()
st = torch.cuda.Stream()
ref = None
for val in sys.argv[3:]:
    if val == "-":
        os.environ.pop(var, None)
    else:
        os.environ[var] = val
    ts = []
    for r in range(6):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):
            e0.record(st)
            g = eh.Graph(s, d, stream=st)
            e1.record(st)
            st.synchronize()
            c = g.count_triangles() if r == 0 else None
            g.close()
        if r:
            ts.append(e0.elapsed_time(e1))
        else:
            t = c
    ref = ref or t
    print(name, var, val, f"load {statistics.median(ts):.3f} ms", "ok" if t == ref else "MISMATCH", flush=True)
