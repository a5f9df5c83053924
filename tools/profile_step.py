"""Profiling driver (development only): M31 N (default 2^23), init + S all-active full steps."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1811_02761_b200 as g2
from paper_1811_02761_b200.gravitree import sample_model
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 23
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
dacc = 2.0 ** -float(sys.argv[3]) if len(sys.argv) > 3 else 2.0 ** -9
m, p, v = sample_model("m31", n, 1)
sim = g2.Simulation(g2.ParticleSystem(m, p, v), g2.GravParams(1.0, 2.0 ** -5, dacc),
                    g2.StepScheme(adaptive=False), g2.EngineConfig())
sim.set_rebuild_every_step(True)
sim.init()
for _ in range(steps):
    r = sim.step()
    print(r.timings, r.events, flush=True)
