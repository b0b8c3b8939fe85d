"""Dev aid: eh_count_batch throughput (input edges/s, pinned host inputs) vs lanes."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1503_02368_b200 as eh  # noqa: E402
import synth  # noqa: E402

name = sys.argv[1]
K = int(sys.argv[2]) if len(sys.argv) > 2 else 8
q = os.environ.get("QUERY", "triangles")
src, dst = synth.CONFIGS[name].generate()
hs = torch.from_numpy(src.view(np.int32)).pin_memory()
hd = torch.from_numpy(dst.view(np.int32)).pin_memory()
lists = [(hs, hd)] * K
for lanes in sys.argv[3:] or ["1", "2"]:
    os.environ["EH_TEST_BATCH_LANES"] = lanes
    eh.count_batch(lists[:4], q)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    legacy = torch.cuda.default_stream()
    e0.record(legacy)
    t0 = time.perf_counter()
    c = eh.count_batch(lists, q)
    t1 = time.perf_counter()
    e1.record(legacy)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / K
    print(name, q, "lanes", lanes, f"{ms:.3f} ms/step (host {1e3 * (t1 - t0) / K:.3f})",
          f"{src.size / ms / 1e6:.3e} input edges/s", len(set(c)) == 1, flush=True)
