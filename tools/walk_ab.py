"""A/B timing of library builds (development only).

usage: python tools/walk_ab.py N LIB1 [LIB2 ...]  -> mean phase times per build, M31 all-active steps
       G2_AB_PAPER=1 python tools/walk_ab.py ...  -> paper protocol (dt_max 1, rebuild every 2), 32 steps
Each build runs in its own subprocess (G2_LIB_PATH) on the same input."""
import json, os, subprocess, sys

if len(sys.argv) > 2 and sys.argv[1] != "--child":
    n = sys.argv[1]
    for lib in sys.argv[2:]:
        env = dict(os.environ, G2_LIB_PATH=os.path.abspath(lib))
        out = subprocess.run([sys.executable, __file__, "--child", n], env=env, capture_output=True, text=True)
        print(lib, out.stdout.strip() or out.stderr[-2000:], flush=True)
    sys.exit(0)

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import paper_1811_02761_b200 as g2  # noqa: E402
from paper_1811_02761_b200.gravitree import sample_model  # noqa: E402

n = int(sys.argv[2])
m, p, v = sample_model("m31", n, 1)
if os.environ.get("G2_AB_PAPER"):
    sim = g2.Simulation(g2.ParticleSystem(m, p, v), g2.GravParams(1.0, 2.0 ** -5, 2.0 ** -9),
                        g2.StepScheme(dt_max=1.0), g2.EngineConfig())
    sim.init()
    sim.set_fixed_rebuild_interval(2)
    for _ in range(4):
        sim.step()
    rs = [sim.step() for _ in range(32)]
    tot = [r.timings.total() for r in rs]
    small = [r.timings.walk_tree for r in rs if r.active < 0.03 * n]
    print(json.dumps({"paper_ms_per_step": round(1e3 * float(np.mean(tot)), 3),
                      "walk_ms_per_step": round(1e3 * float(np.mean([r.timings.walk_tree for r in rs])), 3),
                      "small_walk_ms": round(1e3 * float(np.mean(small)), 3) if small else None}))
    sys.exit(0)
sim = g2.Simulation(g2.ParticleSystem(m, p, v), g2.GravParams(1.0, 2.0 ** -5, 2.0 ** -9),
                    g2.StepScheme(adaptive=False), g2.EngineConfig())
sim.set_rebuild_every_step(True)
sim.init()
for _ in range(3):
    sim.step()
rs = [sim.step() for _ in range(6)]
keys = vars(rs[0].timings).keys()
res = {k: round(1e3 * float(np.mean([getattr(r.timings, k) for r in rs])), 3) for k in keys}
res["walk_tflops"] = round(g2.walk_flops(rs[-1].events) / (res["walk_tree"] * 1e-3) / 1e12, 2)
print(json.dumps(res))
