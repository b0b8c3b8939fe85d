"""Design aid (not product, not oracle): statistics of the degree-oriented
rank-space CSR of a config, used to choose kernel dispatch thresholds.
numpy only; prints cost-model sums over oriented edges."""
import sys, time
import numpy as np
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import synth

def build(src, dst):
    s = src.astype(np.uint64); d = dst.astype(np.uint64)
    k = s != d
    lo = np.minimum(s[k], d[k]); hi = np.maximum(s[k], d[k])
    key = np.unique((lo << 32) | hi)
    u = (key >> 32).astype(np.int64); v = (key & 0xffffffff).astype(np.int64)
    n = int(max(u.max(), v.max())) + 1
    deg = np.bincount(u, minlength=n) + np.bincount(v, minlength=n)
    act = np.nonzero(deg)[0]
    order = act[np.lexsort((act, deg[act]))]
    rank = np.full(n, -1, np.int64); rank[order] = np.arange(order.size)
    ru, rv = rank[u], rank[v]
    a = np.minimum(ru, rv); b = np.maximum(ru, rv)
    o = np.lexsort((b, a)); a = a[o]; b = b[o]
    nact = order.size
    dplus = np.bincount(a, minlength=nact)
    rp = np.zeros(nact + 1, np.int64); rp[1:] = np.cumsum(dplus)
    return nact, rp, a, b, dplus

def main(cfg):
    t = time.time()
    src, dst = synth.CONFIGS[cfg].generate()
    nact, rp, ex, ey, dplus = build(src, dst)
    m = ex.size
    print(f"{cfg}: m={m} nact={nact} max d+={dplus.max()} build {time.time()-t:.1f}s")
    first = np.where(dplus > 0, ey[np.minimum(rp[:-1], m-1)], 0)
    last = np.where(dplus > 0, ey[np.maximum(rp[1:]-1, 0)], 0)
    span = np.where(dplus > 0, last - first + 1, 0)
    for tau in (32, 256):
        dense = (dplus > 0) & (span < tau * dplus)
        words = np.where(dense, (last >> 5) - (first >> 5) + 1, 0)
        print(f" tau={tau}: dense sets {dense.sum()} elems {dplus[dense].sum()} ({dplus[dense].sum()/m:.3f})")
    tau = 32
    dense = (dplus > 0) & (span < tau * dplus)
    words = np.where(dense, (last >> 5) - (first >> 5) + 1, 0)
    bytes_y = np.where(dense, 4 * words, 4 * dplus)
    # per edge quantities
    pos = np.arange(m) - rp[ex]             # index of y within N+(x)
    asuf = dplus[ex] - 1 - pos              # |N+(x) after y|
    b = dplus[ey]
    W = b.sum()
    print(f" W+ = {W:.3e}  sum a = {asuf.sum():.3e}  sum d+^2 = {(dplus.astype(np.float64)**2).sum():.3e}")
    By = bytes_y[ey].sum()
    Bx = bytes_y.sum()
    print(f" B_tri(32) = {(8*(nact+1) + Bx + By)/1e9:.2f} GB  (y-side {By/1e9:.2f} GB)")
    print(f" edges with b=0: {(b==0).mean():.3f}; a=0: {(asuf==0).mean():.3f}; both>0: {((b>0)&(asuf>0)).mean():.3f}")
    # min-property costs (elements)
    cost_min = np.minimum(asuf, b)
    print(f" sum min(a,b) = {cost_min.sum():.3e}")
    ywords = np.where(dense[ey], words[ey], b)   # stream-y cost in 32-bit words
    print(f" sum stream-y words (layout-aware) = {ywords.sum():.3e}; sum min(a, stream-y) = {np.minimum(asuf, ywords).sum():.3e}")
    # x with d+ < 2 contribute nothing
    print(f" x with d+>=2: {(dplus>=2).sum()}  edges from them {dplus[dplus>=2].sum()}")
    # distribution of x span in words for dense/sparse x
    xw = (last >> 5) - (first >> 5) + 1
    for lim in (256, 1024, 4096, 16384):
        sel = (dplus >= 2) & (xw <= lim)
        print(f"  x span words <= {lim}: {sel.sum()} vertices, edges {dplus[sel].sum()/m:.3f}, W {b[np.isin(ex, np.nonzero(sel)[0])].sum()/W:.3f}")
    # degree histogram of d+
    for lo_, hi_ in [(2, 8), (8, 32), (32, 128), (128, 512), (512, 1 << 30)]:
        sel = (dplus >= lo_) & (dplus < hi_)
        e_sel = np.isin(ex, np.nonzero(sel)[0])
        print(f"  d+ in [{lo_},{hi_}): {sel.sum()} x, edges {e_sel.mean():.3f}, stream-y words {ywords[e_sel].sum():.2e}, sum a {asuf[e_sel].sum():.2e}, min {np.minimum(asuf, ywords)[e_sel].sum():.2e}")
    # dense y share
    print(f" edges with dense y: {dense[ey].mean():.3f}; with dense x: {dense[ex].mean():.3f}")
    # in-degree of y hubs
    dminus = np.bincount(ey, minlength=nact)
    top = np.argsort(-dminus)[:5]
    print(" top d- :", [(int(t), int(dminus[t]), int(dplus[t]), bool(dense[t]), int(words[t])) for t in top])

if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "C2")
