"""Profiling driver: load one config `--reps` times (device-resident inputs)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch  # noqa: E402
import synth  # noqa: E402
import paper_1503_02368_b200 as eh  # noqa: E402
ap = argparse.ArgumentParser(); ap.add_argument("--config", default="C3"); ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
src, dst = synth.CONFIGS[a.config].generate()
s = torch.from_numpy(src.view(np.int32)).cuda(); d = torch.from_numpy(dst.view(np.int32)).cuda()
for _ in range(a.reps):
    with eh.Graph(s, d) as g:
        print(g.stats().m_undirected, flush=True)
