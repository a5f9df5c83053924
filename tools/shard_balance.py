"""Per-group walk cost from a G2_WALK_TRACE file (development): imbalance of contiguous equal-count
group shards over W ranks (the multi-GPU partition) vs cost-balanced shards."""
import sys
import numpy as np
a = np.fromfile(sys.argv[1], dtype=np.uint32).reshape(-1, 8)
grp, macs, pushes = a[:, 4].astype(np.int64), a[:, 6].astype(np.float64), a[:, 7].astype(np.float64)
ng = int(grp.max()) + 1
cost = np.bincount(grp, weights=pushes * 32 * 9 + macs * 30, minlength=ng)  # ~instructions (flush + traversal)
tot = cost.sum()
for W in (2, 4, 8):
    edges = (np.arange(W + 1) * ng) // W
    sh = np.array([cost[edges[r]:edges[r + 1]].sum() for r in range(W)])
    c = np.cumsum(cost)
    bal = np.searchsorted(c, np.arange(1, W) * tot / W)
    e2 = np.concatenate([[0], bal, [ng]])
    sh2 = np.array([cost[e2[r]:e2[r + 1]].sum() for r in range(W)])
    print(f"W={W}: equal-count max/mean {sh.max() / sh.mean():.3f}   cost-balanced max/mean {sh2.max() / sh2.mean():.3f}")
