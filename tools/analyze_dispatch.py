"""Design aid: emulate count_tri.cu's per-row dispatch on a config and report
work units per (class, kind).  numpy; mirrors row_kind()/build_xset()."""
import sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from analyze_workload import build
import synth
cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
tau = int(sys.argv[2]) if len(sys.argv) > 2 else 128
WMAX, WBM, CBM, ANDF = 128, 512 * 32, 16384 * 32, 8
src, dst = synth.CONFIGS[cfg].generate()
nact, rp, ex, ey, dplus = build(src, dst)
m = ex.size
first = np.where(dplus > 0, ey[np.minimum(rp[:-1], m - 1)], 0)
last = np.where(dplus > 0, ey[np.maximum(rp[1:] - 1, 0)], 0)
span = last - first + 1
dense = (dplus >= 2) & (span < tau * dplus)
c0 = first >> 7; c1 = np.where(dense, (last >> 7) + 1, c0)
pos = np.arange(m) - rp[ex]
a = dplus[ex] - 1 - pos
b = dplus[ey]
xd = dplus[ex]
cls = np.where(xd <= WMAX, 0, 1)
xspan_bits = ((last[ex] >> 7) + 1 - (first[ex] >> 7)) * 128
xbm = np.where(cls == 0, xspan_bits <= WBM, xspan_bits <= CBM)
live = (a > 0) & (b > 0)
yden = dense[ey]
xc0 = first[ex] >> 7; xc1 = (last[ex] >> 7) + 1
ov = np.minimum(c1[ey], xc1) - np.maximum(c0[ey], xc0)
kind = np.full(m, 0)
kd_dense = live & yden
skip_and = kd_dense & xbm & (ov <= 0)
use_and = kd_dense & xbm & (ov > 0) & (ov <= ANDF * a + 8)
probe = kd_dense & ~skip_and & ~use_and
lg = np.floor(np.log2(np.maximum(b, 1))) + 1
search = live & ~yden & (a * lg * 4 < b)
stream = live & ~yden & ~search
for c in (0, 1):
    sel = cls == c
    print(f"{cfg} tau={tau} class {'warp' if c == 0 else 'cta'}: x {len(np.unique(ex[sel]))} rows {sel.sum()} live {(live&sel).sum()} xbm-rows {(xbm&sel&live).sum()}")
    print(f"   probe rows {(probe&sel).sum():>10} units(a) {a[probe&sel].sum():.3e}  rows<32: {(probe&sel&(a<32)).sum()}")
    print(f"   and   rows {(use_and&sel).sum():>10} units(ch) {ov[use_and&sel].sum():.3e}  rows<32: {(use_and&sel&(ov<32)).sum()}")
    print(f"   strm  rows {(stream&sel).sum():>10} units(b) {b[stream&sel].sum():.3e}  rows<128: {(stream&sel&(b<128)).sum()} hash-x rows {(stream&sel&~xbm).sum()}")
    print(f"   srch  rows {(search&sel).sum():>10} units(a) {a[search&sel].sum():.3e} (x log b {(a*lg)[search&sel].sum():.3e})")
