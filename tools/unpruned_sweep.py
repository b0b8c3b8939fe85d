"""Dev aid: time eh_count_triangles_unpruned on one config under several values of an
environment switch ("-" = unset)."""
import os
import statistics
import sys
import time

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
with eh.Graph(s, d) as g:
    t = g.count_triangles()
    g.count_triangles_unpruned()  # builds the symmetric trie
    for val in sys.argv[3:]:
        if val == "-":
            os.environ.pop(var, None)
        else:
            os.environ[var] = val
        ts = []
        for r in range(4):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            c = g.count_triangles_unpruned()
            ts.append((time.perf_counter() - t0) * 1e3)
        print(name, var, val, f"{statistics.median(ts[1:]):.2f} ms", "ok" if c == 6 * t else "MISMATCH", flush=True)
