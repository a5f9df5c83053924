"""Per-rank walk work of in-process meshes (development): equal-count shards (copy mesh) vs the
cost-balanced shards of the fused peer exchange, M31 N all-active, rebuild every step."""
import os, sys, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1811_02761_b200 as g2
from paper_1811_02761_b200.gravitree import sample_model
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 22
m, p, v = sample_model("m31", n, 1)
for world in (2, 4, 8):
    for mesh in ("copy", "p2p"):
        sims = []
        for _ in range(world):
            s = g2.Simulation(g2.ParticleSystem(m, p, v), g2.GravParams(1.0, 2.0 ** -5, 2.0 ** -9),
                              g2.StepScheme(dt_max=1 / 16, adaptive=False))
            s.set_rebuild_every_step(True)
            sims.append(s)
        (g2.Simulation.set_mesh_local if mesh == "copy" else g2.Simulation.set_mesh_local_p2p)(sims)
        for s in sims:
            s.init()
        for _ in range(3):
            out = [None] * world
            th = [threading.Thread(target=lambda k: out.__setitem__(k, sims[k].step()), args=(k,)) for k in range(world)]
            [t.start() for t in th]
            [t.join() for t in th]
        w = np.array([o.events.interactions for o in out], float)
        print(f"N={n} world={world} {mesh:4s} max/mean interactions {w.max() / w.mean():.4f}", flush=True)
        del sims
