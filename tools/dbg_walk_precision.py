import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_1811_02761_b200 as g2
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
g = np.load("tests/golden/m31_16384.npz")
s = g2.ParticleSystem(g["mass"], g["pos"], acc_old_mag=g["acc_old_mag"])
eng = g2.GravityEngine(g2.GravParams(1.0, 2.0 ** -5, 2.0 ** -9))
eng.build(s); ev = eng.evaluate(s)
a, r = s.acc, g["acc"]
e = np.linalg.norm(a - r, axis=1) / np.linalg.norm(r, axis=1)
rad = np.linalg.norm(g["pos"], axis=1)
print("max |x|", np.abs(g["pos"]).max(), "mass range", g["mass"].min(), g["mass"].max())
for lo, hi in [(0, 1), (1, 5), (5, 20), (20, 100), (100, 1e9)]:
    m = (rad >= lo) & (rad < hi)
    if m.any(): print(f"r in [{lo},{hi}): n={m.sum()} median {np.median(e[m]):.2e} p99 {np.quantile(e[m], .99):.2e}")
t = eng.tree()
# per-particle error vs position in morton order
er = e[t.perm]
print("morton-order error deciles:", [f"{np.median(er[i*1638:(i+1)*1638]):.1e}" for i in range(10)])
# scaled plummer check
sys.exit(0)
for scale in [1.0, 100.0]:
    mass, pos, _ = plummer(16384, seed=2)
    pos = pos * scale
    s2 = g2.ParticleSystem(mass, pos, acc_old_mag=np.full(16384, 1.0 / scale**2))
    e2 = g2.GravityEngine(g2.GravParams(1.0, 2.0 ** -5 * scale, 2.0 ** -9)); e2.build(s2); e2.evaluate(s2)
    from oracle.refpy import Oracle
    ao, _, _ = Oracle().evaluate(mass, pos, np.full(16384, 1.0 / scale**2), eps=2.0 ** -5 * scale, dacc=2.0 ** -9)
    print("plummer scale", scale, g2.force_error(s2.acc, ao))
