"""Rebuild-tuner trace of a block-step run (development): M31 N, StepScheme(dt_max), the tuner on the
deterministic model clock (flop rate, build seconds per particle) or CUDA events (rate 0); per step the
active fraction, rebuild flag, tuner interval and walk time.
usage: python tools/tuner_trace.py N dt_max steps rate build_per_particle"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1811_02761_b200 as g2
from paper_1811_02761_b200.gravitree import sample_model
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 23
dt_max = float(eval(sys.argv[2])) if len(sys.argv) > 2 else 1.0 / 16
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 36
rate = float(sys.argv[4]) if len(sys.argv) > 4 else 3.8e13
bpp = float(sys.argv[5]) if len(sys.argv) > 5 else 1.8e-10
m, p, v = sample_model("m31", n, 1)
sim = g2.Simulation(g2.ParticleSystem(m, p, v), g2.GravParams(1.0, 2.0 ** -5, 2.0 ** -9), g2.StepScheme(eta=0.5, dt_max=dt_max))
sim.init()
if rate > 0:
    sim.set_tuner_model(rate, bpp)
tot = 0.0
for k in range(steps):
    r = sim.step()
    tot += r.timings.total()
    print(f"{k:3d} act {r.active / n:6.3f} rebuilt {int(r.rebuilt)} interval {r.rebuild_interval:3d} "
          f"walk {r.timings.walk_tree * 1e3:7.2f} ms int/active {r.events.interactions / max(r.active, 1):8.0f}", flush=True)
print(f"mean device s/step {tot / steps:.5f}")
