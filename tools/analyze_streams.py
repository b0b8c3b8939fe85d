"""Design aid: for the warp-class STREAM rows (sparse y, tau=128), how much
re-streaming of the same y happens (candidates for y-major processing)."""
import sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from analyze_workload import build
import synth
cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
tau = 128
src, dst = synth.CONFIGS[cfg].generate()
nact, rp, ex, ey, dplus = build(src, dst)
m = ex.size
first = np.where(dplus > 0, ey[np.minimum(rp[:-1], m - 1)], 0)
last = np.where(dplus > 0, ey[np.maximum(rp[1:] - 1, 0)], 0)
span = last - first + 1
dense = (dplus >= 2) & (span < tau * dplus)
pos = np.arange(m) - rp[ex]
a = dplus[ex] - 1 - pos
b = dplus[ey]
lg = np.floor(np.log2(np.maximum(b, 1))) + 1
live = (a > 0) & (b > 0)
warp = dplus[ex] <= 128
stream = live & ~dense[ey] & ~(a * lg * 4 < b)
for name, sel in (("warp", stream & warp), ("cta", stream & ~warp)):
    ys = ey[sel]
    uy, cnt = np.unique(ys, return_counts=True)
    print(f"{cfg} {name}: stream rows {sel.sum()}, distinct y {uy.size}, sum b {b[sel].sum():.3e}, "
          f"sum_y b once {dplus[uy].sum():.3e}, sum a {a[sel].sum():.3e}")
    for lo, hi in ((1, 2), (2, 8), (8, 64), (64, 10**9)):
        k = (cnt >= lo) & (cnt < hi)
        print(f"   y streamed [{lo},{hi}) times: {k.sum()} ys, rows {cnt[k].sum()}, sum b {(dplus[uy[k]] * cnt[k]).sum():.3e}")
    # distribution of a and b on stream rows
    print("   a pct", np.percentile(a[sel], [50, 90, 99]), " b pct", np.percentile(b[sel], [50, 90, 99]))
