"""Design aid: for STREAM rows (sparse y, warp class), the share of N+(y) that
lies inside [min A, max A] (A = N+(x) after y)."""
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
stream = live & ~dense[ey] & ~(a * lg * 4 < b) & warp
idx = np.nonzero(stream)[0]
amin = ey[np.minimum(idx + 1, m - 1)]
amax = last[ex[idx]]
yy = ey[idx]
# count N+(y) elements in [amin, amax]: global sorted ey within each row segment
lo = np.empty(idx.size, np.int64); hi = np.empty(idx.size, np.int64)
chunk = 1 << 22
for s in range(0, idx.size, chunk):
    sl = slice(s, s + chunk)
    st = rp[yy[sl]]; en = rp[yy[sl] + 1]
    # vectorised per-row searchsorted via offsetting: use global key = row*2^32 + value
    key_base = yy[sl].astype(np.int64) << 32
    allkeys = (ex.astype(np.int64) << 32) | ey.astype(np.int64)
    lo[sl] = np.searchsorted(allkeys, key_base | amin[sl]) - st
    hi[sl] = np.searchsorted(allkeys, key_base | amax[sl], side="right") - st
inwin = (hi - lo).clip(min=0)
print(f"{cfg}: warp STREAM rows {idx.size}, sum b {b[idx].sum():.3e}, sum in-window {inwin.sum():.3e} "
      f"({inwin.sum() / b[idx].sum():.3f})")
