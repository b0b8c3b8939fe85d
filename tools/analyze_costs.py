"""Design aid: per-edge cost classes for the triangle kernel (numpy)."""
import sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from analyze_workload import build
import synth
cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
src, dst = synth.CONFIGS[cfg].generate()
nact, rp, ex, ey, dplus = build(src, dst)
m = ex.size
first = np.where(dplus > 0, ey[np.minimum(rp[:-1], m - 1)], 0)
last = np.where(dplus > 0, ey[np.maximum(rp[1:] - 1, 0)], 0)
span = np.where(dplus > 0, last - first + 1, 0)
pos = np.arange(m) - rp[ex]
a = dplus[ex] - 1 - pos
b = dplus[ey]
live = (a > 0) & (b > 0)
print(f"{cfg}: m={m}, live edges {live.sum()} ({live.mean():.3f})")
for tau in (32, 64, 256):
    dense = (dplus >= 2) & (span < tau * dplus)
    bsbytes = np.where(dense, ((last >> 7) - (first >> 7) + 1) * 16, 0)
    yd = dense[ey] & live
    ys = (~dense[ey]) & live
    print(f" tau={tau}: dense sets {dense.sum()}, pool {bsbytes.sum()/1e6:.1f} MB; live edges dense-y {yd.sum()} sparse-y {ys.sum()}")
    print(f"   dense-y: sum a {a[yd].sum():.3e}  sum b {b[yd].sum():.3e}  sum ychunks {(bsbytes[ey][yd]/16).sum():.3e}")
    lb = np.log2(np.maximum(b, 2))
    print(f"   sparse-y: sum a {a[ys].sum():.3e}  sum b {b[ys].sum():.3e}  sum a*log2b {(a*lb)[ys].sum():.3e}  sum min(b, a*log2b) {np.minimum(b, a*lb)[ys].sum():.3e} sum min(a,b) {np.minimum(a,b)[ys].sum():.3e}")
    # small-x share
    for lo, hi in ((2, 33), (33, 10**9)):
        sx = (dplus[ex] >= lo) & (dplus[ex] < hi)
        print(f"   x d+ in [{lo},{hi}): live {(live&sx).sum()} dense-y {(yd&sx).sum()} sparse-y sum b {b[ys&sx].sum():.2e} sum a {a[ys&sx].sum():.2e} min {np.minimum(b, a*lb)[ys&sx].sum():.2e}")
