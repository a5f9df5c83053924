"""In-process fused-exchange mesh probe (development): world Simulations on one device, M31 N,
three sharded all-active steps; prints each rank's walk events per step.

usage: python tools/p2p_local_probe.py N WORLD"""
import os, sys, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1811_02761_b200 as g2
from paper_1811_02761_b200.gravitree import sample_model
n = int(sys.argv[1]); world = int(sys.argv[2])
m, p, v = sample_model("m31", n, 1)
sims = []
for _ in range(world):
    s = g2.Simulation(g2.ParticleSystem(m, p, v), g2.GravParams(1.0, 2.0 ** -5, 2.0 ** -9), g2.StepScheme(dt_max=1 / 16, adaptive=False))
    s.set_rebuild_every_step(True); sims.append(s)
g2.Simulation.set_mesh_local_p2p(sims)
for s in sims: s.init()
print("init done", flush=True)
for k in range(3):
    out = [None] * world
    th = [threading.Thread(target=lambda j: out.__setitem__(j, sims[j].step()), args=(j,)) for j in range(world)]
    [t.start() for t in th]; [t.join() for t in th]
    print("step", k, [o.events.interactions for o in out], flush=True)
