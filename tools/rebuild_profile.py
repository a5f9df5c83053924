"""Rebuild-step profile (development): M31 N (default 2^23) block steps with a rebuild every step;
prints per-step phase times and the Simulation's sort statistics (bucket sorts / radix fallbacks)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1811_02761_b200 as g2
from paper_1811_02761_b200.gravitree import sample_model
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 23
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
m, p, v = sample_model("m31", n, 1)
sim = g2.Simulation(g2.ParticleSystem(m, p, v), g2.GravParams(1.0, 2.0 ** -5, 2.0 ** -9), g2.StepScheme(dt_max=1.0))
sim.init()
sim.set_fixed_rebuild_interval(1)
for k in range(steps):
    r = sim.step()
    t = r.timings
    print(f"{k} act {r.active / n:.3f} rebuilt {int(r.rebuilt)} predict {t.predict * 1e3:.3f} make_tree {t.make_tree * 1e3:.3f} "
          f"calc_node {t.calc_node * 1e3:.3f} walk {t.walk_tree * 1e3:.3f} ms", flush=True)
print("sort stats (bucket sorts, radix fallbacks):", sim.sort_stats())
