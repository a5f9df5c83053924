"""Per-step walk timelines of the block-step protocol (development): M31 N, dt_max = 1, fixed
rebuild interval 2; run with G2_WALK_TRACE=<dir>/trace.bin and each step's trace is kept as
<dir>/trace_<step>.bin (summarise with tools/trace_stats.py)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1811_02761_b200 as g2
from paper_1811_02761_b200.gravitree import sample_model
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 23
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 8
path = os.environ["G2_WALK_TRACE"]
m, p, v = sample_model("m31", n, 1)
sim = g2.Simulation(g2.ParticleSystem(m, p, v), g2.GravParams(1.0, 2.0 ** -5, 2.0 ** -9), g2.StepScheme(dt_max=1.0))
sim.init()
sim.set_fixed_rebuild_interval(2)
for k in range(steps):
    r = sim.step()
    os.replace(path, path.replace(".bin", f"_{k}.bin"))
    print(k, r.active, r.rebuilt, f"walk {r.timings.walk_tree*1e3:.3f} ms", flush=True)
