"""Quick timing probe (development only): build + walk at a given size."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1811_02761_b200 as g2
from oracle.refpy import Ref

model = sys.argv[1] if len(sys.argv) > 1 else "m31"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 20
t = time.time()
m, p, v = Ref().sample_model(model, n, 1)
print(f"ic {time.time()-t:.1f}s", flush=True)
eng = g2.GravityEngine(g2.GravParams(1.0, 2.0 ** -5, 2.0 ** -9))
s = g2.ParticleSystem(m, p)
t = time.time(); ev0 = eng.bootstrap(s); print(f"bootstrap {time.time()-t:.2f}s {ev0}", flush=True)
for it in range(3):
    t = time.time(); eng.build(s); tb = time.time() - t
    t = time.time(); ev = eng.evaluate(s); tw = time.time() - t
    print(f"build {tb*1e3:.1f} ms  evaluate(host API) {tw*1e3:.1f} ms  {ev}  walk GF/s(host) {g2.walk_flops(ev)/tw/1e9:.0f}", flush=True)
