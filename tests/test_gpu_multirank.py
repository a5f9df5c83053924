"""GPU: the sharded multi-rank step on one device.

Ranks shard the sink groups and exchange accelerations through the same
window/unpack path the NCCL mesh uses (LocalExchange transport).  The
sharded run must equal the single-rank run: identical trees (redundant,
deterministic builds), summed events identical, accelerations equal to
FP32 summation-order tolerance."""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_steps_match_single_rank(world):
    import paper_1811_02761_b200 as g2
    from paper_1811_02761_b200.gravitree import sample_model
    m, p, v = sample_model("m31", 100000, 5)
    params = g2.GravParams(1.0, 2.0 ** -5, 2.0 ** -9)
    scheme = g2.StepScheme(dt_max=1.0 / 64, adaptive=False)

    def make():
        s = g2.Simulation(g2.ParticleSystem(m, p, v), params, scheme)
        s.set_rebuild_every_step(True)
        return s

    ref = make()
    ref.init()
    sims = [make() for _ in range(world)]
    g2.Simulation.set_mesh_local(sims)
    for s in sims:
        s.init()
    for _ in range(3):
        r0 = ref.step()
        out = [None] * world

        def run(k):
            out[k] = sims[k].step()

        th = [threading.Thread(target=run, args=(k,)) for k in range(world)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        assert all(o is not None for o in out)
        assert sum(o.events.interactions for o in out) == r0.events.interactions
        assert sum(o.events.mac_evals for o in out) == r0.events.mac_evals
        assert all(o.active == r0.active for o in out)
    a = ref.system()
    for s in sims:
        b = s.system()
        err = g2.force_error(b.acc, a.acc)
        assert err["median"] <= 1e-6 and err["p99"] <= 1e-5, err
        assert np.max(np.abs(b.pos - a.pos)) < 1e-7  # FP32-order differences, integrated 3 steps
