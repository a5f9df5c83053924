"""Block-step protocol trace (development): per-step active fraction, rebuilds, walk time,
interactions/particle and tuner interval for M31 N with dt_max = 1."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1811_02761_b200 as g2
from paper_1811_02761_b200.gravitree import sample_model
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 23
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 64
fixed = int(sys.argv[3]) if len(sys.argv) > 3 else 0
m, p, v = sample_model("m31", n, 1)
sim = g2.Simulation(g2.ParticleSystem(m, p, v), g2.GravParams(1.0, 2.0 ** -5, 2.0 ** -9), g2.StepScheme(dt_max=1.0))
sim.init()
if fixed:
    sim.set_fixed_rebuild_interval(fixed)
tot = 0.0
ph = dict(walk_tree=0.0, calc_node=0.0, make_tree=0.0, predict=0.0, correct=0.0)
for k in range(steps):
    r = sim.step()
    t = r.timings
    tot += t.total()
    for key in ph:
        ph[key] += getattr(t, key)
    print(f"{k:3d} act {r.active/n:6.3f} rebuilt {int(r.rebuilt)} interval {r.rebuild_interval:3d} walk {t.walk_tree*1e3:8.2f} ms "
          f"build {(t.make_tree+t.calc_node)*1e3:6.2f} ms int/active {r.events.interactions/max(r.active,1):9.0f}", flush=True)
print(f"mean device s/step {tot/steps:.5f}  " + " ".join(f"{k} {v/steps*1e3:.3f}ms" for k, v in ph.items()))
