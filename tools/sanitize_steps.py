"""Block steps under compute-sanitizer (development): a small M31 Simulation through rebuilds (bucket
sort, split, calcNode with the side-stream overlap) and block steps."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1811_02761_b200 as g2
from paper_1811_02761_b200.gravitree import sample_model
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 17
m, p, v = sample_model("m31", n, 1)
sim = g2.Simulation(g2.ParticleSystem(m, p, v), g2.GravParams(1.0, 2.0 ** -5, 2.0 ** -9), g2.StepScheme(dt_max=1.0))
sim.init()
sim.set_fixed_rebuild_interval(2)
for k in range(6):
    r = sim.step()
    print(k, r.active, r.rebuilt, flush=True)
