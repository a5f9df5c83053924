"""Config 4 (BASELINE.json configs[3]): M31 at N = 25 x 2^20 (the paper's largest V100 run) and
2^27 on ONE B200: one all-active full step (rebuild), phase times, walk TFLOP/s, device memory in
use, and force errors vs FP64 direct summation on a random sink sample."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1811_02761_b200 as g2  # noqa: E402
from paper_1811_02761_b200.gravitree import direct_sum_targets, sample_model  # noqa: E402

n = int(eval(sys.argv[1])) if len(sys.argv) > 1 else 25 << 20
nsample = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
t0 = time.time()
m, p, v = sample_model("m31", n, 1)
t_ic = time.time() - t0
params = g2.GravParams(1.0, 2.0 ** -5, 2.0 ** -9)
sim = g2.Simulation(g2.ParticleSystem(m, p, v), params, g2.StepScheme(adaptive=False))
sim.set_rebuild_every_step(True)
sim.init()
rs = [sim.step() for _ in range(3)]
r = rs[-1]
import torch  # noqa: E402  (device memory query only)
free, total = torch.cuda.mem_get_info(0)
st = sim.system()
tg = np.sort(np.random.default_rng(3).choice(n, nsample, replace=False)).astype(np.uint32)
ref = direct_sum_targets(g2.ParticleSystem(m, st.pos), tg, params)
err = g2.force_error(st.acc[tg], ref)
t = r.timings
print(json.dumps({"n": n, "ic_s": round(t_ic, 1), "step_ms": round(t.total() * 1e3, 2),
                  "walk_ms": round(t.walk_tree * 1e3, 2), "make_tree_ms": round(t.make_tree * 1e3, 2),
                  "calc_node_ms": round(t.calc_node * 1e3, 2), "interactions_per_particle": r.events.interactions / n,
                  "walk_tflops": round(g2.walk_flops(r.events) / t.walk_tree / 1e12, 2),
                  "device_mem_used_gb": round((total - free) / 1e9, 1), "err_median": err["median"],
                  "err_p99": err["p99"], "err_max": err["max"], "sample": nsample}))
