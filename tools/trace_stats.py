"""Summarise a G2_WALK_TRACE file (development only)."""
import sys
import numpy as np
a = np.fromfile(sys.argv[1], dtype=np.uint32).reshape(-1, 8)
t0 = a[:, 0].astype(np.uint64) | (a[:, 1].astype(np.uint64) << 32)
t1 = a[:, 2].astype(np.uint64) | (a[:, 3].astype(np.uint64) << 32)
grp, root, macs, pushes = a[:, 4], a[:, 5] & 0xff, a[:, 6].astype(np.float64), a[:, 7].astype(np.float64)
ndon, maxlive = (a[:, 5] >> 8) & 0xfff, a[:, 5] >> 20
base = t0.min()
s = (t0 - base) / 1e6
e = (t1 - base) / 1e6
d = e - s
print("tasks", len(a), "span ms %.3f" % e.max(), "initial", (root == 0).sum(), "donated", (root != 0).sum())
tt = np.linspace(0, e.max(), 21)
print("busy warps:", [int(((s <= x) & (e > x)).sum()) for x in tt])
print("task dur ms: p50 %.4f p99 %.3f max %.3f" % (np.median(d), np.quantile(d, .99), d.max()))
for k in np.argsort(-d)[:6]:
    print("  grp %d root %d dur %.3f start %.3f macs %d pushes %d donations %d max live %d" % (
        grp[k], root[k], d[k], s[k], macs[k], pushes[k], ndon[k], maxlive[k]))
A = np.vstack([pushes, macs, np.ones_like(macs)]).T
coef, *_ = np.linalg.lstsq(A, d * 1e3, rcond=None)
print("dur_us ~ %.4f*pushes + %.4f*macs + %.2f" % tuple(coef))
ini = root == 0
print("last initial start %.3f; donated starts: min %.3f median %.3f" % (s[ini].max(), s[~ini].min() if (~ini).any() else -1, np.median(s[~ini]) if (~ini).any() else -1))
W = int(sys.argv[2]) if len(sys.argv) > 2 else 2368  # producer warps of the walk grid
print("sum task time / (span*warps) = %.3f" % (d.sum() / (e.max() * W)))
