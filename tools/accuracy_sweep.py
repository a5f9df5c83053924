"""Config 5: dacc sweep at M31 N (default 2^23): walk time and force error
against direct summation on a random sample of sinks (FP64 on the GPU).

For each dacc: fresh Simulation (bootstrap = geometric walk, as the reference for n > 65536),
one all-active step with a rebuild; walk time and events from the StepResult; errors of the
new accelerations vs direct summation at the same (predicted) positions, reference
nearest-rank semantics (gravity.cpp:67-90)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1811_02761_b200 as g2  # noqa: E402
from paper_1811_02761_b200.gravitree import direct_sum_targets, sample_model  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 23
nsample = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
out_json = sys.argv[3] if len(sys.argv) > 3 else None
m, p, v = sample_model("m31", n, 1)
tg = np.sort(np.random.default_rng(7).choice(n, nsample, replace=False)).astype(np.uint32)
rows = []
for e in (1, 3, 6, 9, 12, 15, 20):
    dacc = 2.0 ** -e
    params = g2.GravParams(1.0, 2.0 ** -5, dacc)
    sim = g2.Simulation(g2.ParticleSystem(m, p, v), params, g2.StepScheme(dt_max=1.0 / 1024, adaptive=False))
    sim.set_rebuild_every_step(True)
    sim.init()
    r = sim.step()
    st = sim.system()
    ref = direct_sum_targets(g2.ParticleSystem(m, st.pos), tg, params)
    err = g2.force_error(st.acc[tg], ref)
    row = {"dacc": f"2^-{e}", "walk_ms": r.timings.walk_tree * 1e3, "step_ms": r.timings.total() * 1e3,
           "interactions_per_particle": r.events.interactions / n,
           "walk_tflops": g2.walk_flops(r.events) / r.timings.walk_tree / 1e12,
           "median": err["median"], "p99": err["p99"], "max": err["max"]}
    rows.append(row)
    print(json.dumps(row), flush=True)
if out_json:
    with open(out_json, "w") as f:
        json.dump({"n": n, "sample": nsample, "rows": rows}, f, indent=1)
