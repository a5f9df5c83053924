"""Config 5: dacc sweep at M31 N (default 2^23) -- the B200 against the reference at the
SAME N, sinks and inputs.

For each dacc:
  * B200 all-active step (fresh Simulation, rebuild, all particles at level 0): walk time, TFLOP/s;
  * accuracy on every S-th whole sink group (default S = 512 -> 16384 sinks at 2^23): the reference
    library (oracle/_ref) and the B200 walk the same groups with the same acc_old_mag (one geometric
    bootstrap on the B200); both are compared with FP64 direct summation (g2_direct_sum_targets) by
    the reference's nearest-rank force_error (gravity.cpp:67-90); events must agree exactly;
  * SURVEY §8c bar: B200 median and p99 <= max(1.05 x reference, reference + 2e-6).

usage: python tools/accuracy_sweep.py [N] [S] [out.json]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1811_02761_b200 as g2  # noqa: E402
from oracle.refpy import Ref  # noqa: E402
from paper_1811_02761_b200.gravitree import direct_sum_targets, sample_model  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 23
every = int(sys.argv[2]) if len(sys.argv) > 2 else 512
out_json = sys.argv[3] if len(sys.argv) > 3 else None
EPS = 2.0 ** -5
ref = Ref()
m, p, v = sample_model("m31", n, 1)
s0 = g2.ParticleSystem(m, p)
g2.GravityEngine(g2.GravParams(1.0, EPS, 2.0 ** -9)).bootstrap(s0)
amag = s0.acc_old_mag.copy()
perm = ref.build_tree(m, p, with_nodes=False).perm
groups = np.arange(0, (n + 31) // 32, every)
idx = (groups[:, None] * 32 + np.arange(32)[None, :]).ravel()
tg = perm[idx[idx < n]].astype(np.uint32)
direct = None
rows = []
for e in (1, 3, 6, 9, 12, 15, 20):
    dacc = 2.0 ** -e
    params = g2.GravParams(1.0, EPS, dacc)
    sim = g2.Simulation(g2.ParticleSystem(m, p, v), params, g2.StepScheme(dt_max=1.0 / 1024, adaptive=False))
    sim.set_rebuild_every_step(True)
    sim.init()
    sim.step()
    r = sim.step()
    if direct is None:
        direct = direct_sum_targets(g2.ParticleSystem(m, p), tg, params)
    eng_r = ref.engine(eps=EPS, dacc=dacc, threads=0)
    eng_r.build(m, p)
    t0 = time.perf_counter()
    acc_r, _, ev_r = eng_r.evaluate(m, p, amag, targets=tg)
    t_ref = time.perf_counter() - t0
    s = g2.ParticleSystem(m, p, acc_old_mag=amag)
    eng = g2.GravityEngine(params)
    eng.build(s)
    ev = eng.evaluate(s, targets=tg)
    eg, er = g2.force_error(s.acc[tg], direct), g2.force_error(acc_r[tg], direct)
    ok = all(eg[q] <= max(1.05 * er[q], er[q] + 2e-6) for q in ("median", "p99"))
    row = {"dacc": f"2^-{e}", "walk_ms": r.timings.walk_tree * 1e3, "step_ms": r.timings.total() * 1e3,
           "interactions_per_particle": r.events.interactions / n,
           "walk_tflops": g2.walk_flops(r.events) / r.timings.walk_tree / 1e12,
           "b200": {k: eg[k] for k in ("median", "p99", "max")}, "reference": {k: er[k] for k in ("median", "p99", "max")},
           "events_equal": (ev.interactions, ev.mac_evals, ev.list_pushes) == (
               ev_r["interactions"], ev_r["mac_evals"], ev_r["list_pushes"]),
           "bar_met": ok, "reference_walk_s_on_sample": t_ref}
    rows.append(row)
    print(json.dumps(row), flush=True)
if out_json:
    with open(out_json, "w") as f:
        json.dump({"n": n, "groups_every": every, "sinks": int(len(tg)), "rows": rows}, f, indent=1)
