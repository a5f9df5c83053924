"""GPU parity at the configurations the claims are made on (BASELINE configs 3-5).

* config 3 (the bench input, M31 N = 2^23, dacc 2^-9): every 32nd sink group of the all-active walk --
  whole groups, exactly the reference's chunks of 32 consecutive Morton ranks (engine.cpp:38-44) --
  walked by the reference library and by the B200 on identical input and acc_old_mag: events exact,
  accelerations within the FP32 bar (median <= 1e-5, p99 <= 1e-4 relative);
* config 5 (dacc sweep at 2^23): on every 512th group (16384 sinks), the reference's own error and the
  B200's error against FP64 direct summation (g2_direct_sum_targets) at the SAME N and sinks; the B200
  meets SURVEY §8c's bar, median and p99 <= max(1.05 x reference, reference + 2e-6);
* config 4 (M31 25 x 2^20, the paper's largest V100 run): the tree equals build_tree bit for bit;
* potentials at config 3 on every 128th group against the reference's;
* the paper block-step protocol at config 3 stepped beside the reference's own Simulation.
"""
import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

N23 = 1 << 23
EPS = 2.0 ** -5
MED_TOL, P99_TOL = 1e-5, 1e-4


@pytest.fixture(scope="module")
def g2():
    import paper_1811_02761_b200 as g2mod
    return g2mod


@pytest.fixture(scope="module")
def m31_23(g2):
    """The bench input and a realistic acc_old_mag (one geometric bootstrap walk on the B200, as the
    reference's bootstrap does for n > 65536, engine.cpp:95-100); both sides get these exact bits."""
    from paper_1811_02761_b200.gravitree import sample_model
    m, p, _ = sample_model("m31", N23, 1)
    s = g2.ParticleSystem(m, p)
    g2.GravityEngine(g2.GravParams(1.0, EPS, 2.0 ** -9)).bootstrap(s)
    return m, p, s.acc_old_mag.copy()


def group_targets(perm, every, gs=32):
    """Original ids of every `every`-th whole group of the all-active walk (ranks g*gs .. g*gs+gs-1)."""
    n = len(perm)
    groups = np.arange(0, (n + gs - 1) // gs, every)
    idx = (groups[:, None] * gs + np.arange(gs)[None, :]).ravel()
    return perm[idx[idx < n]].astype(np.uint32)


def walk_both(g2, ref, m, p, amag, dacc, tg):
    e = ref.engine(eps=EPS, dacc=dacc, threads=0)
    e.build(m, p)
    acc_r, _, ev_r = e.evaluate(m, p, amag, targets=tg)
    s = g2.ParticleSystem(m, p, acc_old_mag=amag)
    eng = g2.GravityEngine(g2.GravParams(1.0, EPS, dacc))
    eng.build(s)
    ev = eng.evaluate(s, targets=tg)
    return s.acc[tg], acc_r[tg], ev, ev_r, eng


def test_config3_sampled_groups_vs_reference(g2, ref, m31_23):
    m, p, amag = m31_23
    rt = ref.build_tree(m, p, with_nodes=False)
    tg = group_targets(rt.perm, 32)
    assert len(tg) == N23 // 32
    acc, acc_r, ev, ev_r, _ = walk_both(g2, ref, m, p, amag, 2.0 ** -9, tg)
    assert (ev.interactions, ev.mac_evals, ev.list_pushes) == (ev_r["interactions"], ev_r["mac_evals"],
                                                               ev_r["list_pushes"])
    err = g2.force_error(acc, acc_r)
    assert err["median"] <= MED_TOL and err["p99"] <= P99_TOL, err


@pytest.mark.parametrize("e", [3, 9, 15])
def test_config5_dacc_sweep_same_n(g2, ref, m31_23, e):
    from paper_1811_02761_b200.gravitree import direct_sum_targets
    m, p, amag = m31_23
    dacc = 2.0 ** -e
    rt = ref.build_tree(m, p, with_nodes=False)
    tg = group_targets(rt.perm, 512)
    acc, acc_r, ev, ev_r, _ = walk_both(g2, ref, m, p, amag, dacc, tg)
    assert (ev.interactions, ev.mac_evals, ev.list_pushes) == (ev_r["interactions"], ev_r["mac_evals"],
                                                               ev_r["list_pushes"])
    direct = direct_sum_targets(g2.ParticleSystem(m, p), tg, g2.GravParams(1.0, EPS, dacc))
    eg, er = g2.force_error(acc, direct), g2.force_error(acc_r, direct)
    for q in ("median", "p99"):
        assert eg[q] <= max(1.05 * er[q], er[q] + 2e-6), (q, eg, er)


def test_config3_potentials_vs_reference(g2, ref, m31_23):
    """Potentials (flush_list<true>, traversal.cpp:61-84, self term excluded only for |d|^2 == 0,
    :78) at the headline N on every 128th whole group: events exact, potentials within the FP32 bar,
    accelerations unchanged by the potential path."""
    m, p, amag = m31_23
    rt = ref.build_tree(m, p, with_nodes=False)
    tg = group_targets(rt.perm, 128)
    e = ref.engine(eps=EPS, dacc=2.0 ** -9, threads=0)
    e.build(m, p)
    acc_r, pot_r, ev_r = e.evaluate(m, p, amag, targets=tg, with_potential=True)
    s = g2.ParticleSystem(m, p, acc_old_mag=amag)
    eng = g2.GravityEngine(g2.GravParams(1.0, EPS, 2.0 ** -9))
    eng.build(s)
    pot = np.zeros(N23)
    ev = eng.evaluate(s, targets=tg, pot_out=pot)
    assert (ev.interactions, ev.mac_evals, ev.list_pushes) == (ev_r["interactions"], ev_r["mac_evals"],
                                                               ev_r["list_pushes"])
    rel = np.abs(pot[tg] - pot_r[tg]) / np.abs(pot_r[tg])
    assert np.median(rel) <= MED_TOL and np.quantile(rel, 0.99) <= P99_TOL, (np.median(rel), np.quantile(rel, 0.99))
    err = g2.force_error(s.acc[tg], acc_r[tg])
    assert err["median"] <= MED_TOL and err["p99"] <= P99_TOL, err


def test_config4_tree_bitexact_25x2e20(g2, ref):
    from paper_1811_02761_b200.gravitree import sample_model
    m, p, _ = sample_model("m31", 25 << 20, 1)
    eng = g2.GravityEngine(g2.GravParams())
    eng.build(g2.ParticleSystem(m, p))
    t = eng.tree()
    rt = ref.build_tree(m, p)
    for k in ("bbox", "keys", "perm", "rank", "cells", "depth", "nodes"):
        assert np.array_equal(getattr(t, k), getattr(rt, k)), k


def test_config3_paper_protocol_steps_vs_reference(g2, ref):
    """The paper-comparable block-step protocol at the headline N (M31 2^23, dt_max = 1, a fixed
    rebuild interval of 2: bench.py's `paper_protocol.rebuild_every_2`) stepped side by side with the
    reference's own Simulation (integrator.cpp:97-164) from the same input: the same steps rebuild,
    the simulated time advances identically, the active sets agree to the few particles whose block
    level sits on a boundary within FP32 force error, every rebuilt tree equals the reference
    build_tree of the GPU's positions bit for bit, and the states stay together (positions and
    velocities within FP32-force-error drift)."""
    from paper_1811_02761_b200.gravitree import sample_model
    m, p, v = sample_model("m31", N23, 1)
    params = g2.GravParams(1.0, EPS, 2.0 ** -9)
    sim = g2.Simulation(g2.ParticleSystem(m, p, v), params, g2.StepScheme(dt_max=1.0))
    sim.init()
    sim.set_fixed_rebuild_interval(2)
    rs = ref.simulation(m, p, v, G=1.0, eps=EPS, dacc=2.0 ** -9, dt_max=1.0, threads=0)
    rs.init()
    rs.set_fixed_rebuild_interval(2)
    rebuilds = 0
    for k in range(8):
        r, rr = sim.step(), rs.step()
        assert bool(r.rebuilt) == rr["rebuilt"], k
        assert abs(r.active - rr["active"]) <= max(64, rr["active"] // 10000), (k, r.active, rr["active"])
        assert sim.time() == rs.state()["time"], k
        if r.rebuilt:
            rebuilds += 1
            t, rt = sim.tree(), ref.build_tree(m, sim.system().pos)
            for key in ("bbox", "keys", "perm", "rank", "cells", "depth"):
                assert np.array_equal(getattr(t, key), getattr(rt, key)), (k, key)
    assert rebuilds == 3  # steps 2, 4, 6 (init built the first tree)
    st, rst = sim.system(), rs.state()
    ext = np.max(np.abs(rst["pos"]))
    dx = np.linalg.norm(st.pos - rst["pos"], axis=1) / ext
    dv = np.linalg.norm(st.vel - rst["vel"], axis=1) / np.median(np.linalg.norm(rst["vel"], axis=1))
    lv = np.count_nonzero(st.level != rst["level"])
    print(f"paper protocol 8 steps: dx/ext median {np.median(dx):.3e} p99 {np.quantile(dx, .99):.3e} "
          f"max {dx.max():.3e}; dv/|v| median {np.median(dv):.3e} p99 {np.quantile(dv, .99):.3e} "
          f"max {dv.max():.3e}; levels differing {lv}")
    # measured on the B200: dx/extent p99 1.7e-8, dv/median|v| p99 4.8e-5 (the velocity kicks carry the
    # FP32 force error, whose own bar is p99 <= 1e-4 of the force), 16 levels differing; no bound on the
    # max (a particle whose level flipped takes a different kick)
    assert np.quantile(dx, 0.99) <= 1e-7 and np.quantile(dv, 0.99) <= 2e-4, (np.quantile(dx, .99), np.quantile(dv, .99))
    assert lv <= max(64, N23 // 10000), lv
