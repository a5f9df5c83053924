"""GPU parity: the sm_100a path (through the C-ABI) against the CPU oracle.

Bars: keys / perm / rank / cells bit-exact; node attributes,
group spheres, bootstrap direct sum and the integrator bit-exact in FP64;
traversal events exact; accelerations FP32-tolerance vs the FP64 oracle:
relative error median <= 1e-5 and p99 <= 1e-4 (MED_TOL / P99_TOL below).
"""
import numpy as np
import pytest

from conftest import load_golden, plummer, random_cloud

pytestmark = pytest.mark.gpu

MED_TOL = 1e-5
P99_TOL = 1e-4


@pytest.fixture(scope="module")
def g2():
    import paper_1811_02761_b200 as g2mod
    return g2mod


def tree_equal(t, ot):
    for k in ("keys", "perm", "rank", "cells", "depth", "nodes"):
        a, b = getattr(t, k), getattr(ot, k)
        assert a.shape == b.shape, (k, a.shape, b.shape)
        assert np.array_equal(a, b), f"{k} differs at {np.argwhere(a != b)[:5]}"
    assert np.array_equal(t.bbox, ot.bbox)


def gpu_tree(g2, mass, pos, leaf_cap=8):
    eng = g2.GravityEngine(g2.GravParams(), g2.EngineConfig(leaf_cap=leaf_cap))
    eng.build(g2.ParticleSystem(mass, pos))
    return eng.tree()


# ---------------------------------------------------------------- tree (makeTree + calcNode)
@pytest.mark.parametrize("n,leaf_cap", [(1, 8), (2, 8), (9, 8), (1000, 8), (4096, 1), (4096, 4), (65536, 8),
                                        (65536, 16), (200000, 8)])
def test_tree_bitexact_plummer(g2, oracle, n, leaf_cap):
    mass, pos, _ = plummer(n, seed=n)
    tree_equal(gpu_tree(g2, mass, pos, leaf_cap), oracle.build_tree(mass, pos, leaf_cap))


@pytest.mark.parametrize("name", ["plummer_4096", "m31_16384"])
def test_tree_bitexact_golden(g2, name):
    g = load_golden(name)
    t = gpu_tree(g2, g["mass"], g["pos"])
    for k in ("keys", "perm", "rank", "cells", "depth", "nodes", "bbox"):
        assert np.array_equal(getattr(t, k), g["tree_" + k]), k


def test_tree_random_cloud_and_invariants(g2, oracle):
    mass, pos, _ = random_cloud(1000, 11)
    t = gpu_tree(g2, mass, pos)
    tree_equal(t, oracle.build_tree(mass, pos))
    leaves = t.cells[:, 1] == 0
    assert t.cells[leaves, 3].sum() == 1000  # test_tree.cpp:105-126
    assert np.all(np.diff(t.keys.astype(np.uint64)) >= 0)
    assert np.array_equal(np.sort(t.perm), np.arange(1000))


def test_tree_octants_and_coincident(g2, oracle):
    pos = np.array([[sx, sy, sz] for sx in (-.25, .25) for sy in (-.25, .25) for sz in (-.25, .25)])
    t = gpu_tree(g2, np.ones(8), pos, leaf_cap=1)  # test_tree.cpp:86-103
    assert len(t.cells) == 9 and t.cells[0, 1] == 8
    pos = np.tile([0.125, 0.125, 0.125], (20, 1))
    pos[19] = [-0.9, 0, 0]
    t = gpu_tree(g2, np.ones(20), pos, leaf_cap=4)  # test_tree.cpp:166-183
    tree_equal(t, oracle.build_tree(np.ones(20), pos, 4))
    assert t.cells[t.cells[:, 1] == 0, 3].max() == 19
    assert t.depth.max() == 21


def test_morton_corners(g2):
    # unit cube at the origin via two corner particles: key(min) == 0, key(max) == 2^63-1 (test_tree.cpp:42-46)
    pos = np.array([[-0.5, -0.5, -0.5], [0.5, 0.5, 0.5]])
    t = gpu_tree(g2, np.ones(2), pos)
    assert int(t.keys[0]) == 0 and int(t.keys[1]) == 0x7fffffffffffffff


def test_refresh_stale_topology(g2, oracle):
    mass, pos, _ = plummer(20000, seed=5)
    rng = np.random.default_rng(3)
    moved = pos + rng.uniform(-0.05, 0.05, pos.shape)
    eng = g2.GravityEngine(g2.GravParams(), g2.EngineConfig())
    eng.build_structure(g2.ParticleSystem(mass, pos))
    eng.refresh(g2.ParticleSystem(mass, moved))
    t = eng.tree()
    ot = oracle.calc_node_on(mass, pos, mass, moved)
    assert np.array_equal(t.nodes, ot.nodes)
    assert np.array_equal(t.cells, ot.cells)


def test_nonfinite_rejected(g2):
    mass, pos, _ = plummer(100)
    pos[7, 1] = np.nan
    eng = g2.GravityEngine()
    with pytest.raises(g2.DataError):
        eng.build(g2.ParticleSystem(mass, pos))


# ---------------------------------------------------------------- walk (walkTree)
def walk_case(g2, oracle, mass, pos, am, p, cfg=None, targets=None, pot=False):
    cfg = cfg or g2.EngineConfig()
    s = g2.ParticleSystem(mass, pos, acc_old_mag=am)
    eng = g2.GravityEngine(p, cfg)
    eng.build(s)
    pot_g = np.zeros(len(mass)) if pot else None
    ev = eng.evaluate(s, targets=targets, pot_out=pot_g)
    acc_o, pot_o, ev_o = oracle.evaluate(mass, pos, am, targets=targets, G=p.G, eps=p.eps, dacc=p.dacc,
                                         leaf_cap=cfg.leaf_cap, group_size=cfg.group_size, theta=cfg.bootstrap_theta,
                                         with_potential=pot)
    assert (ev.interactions, ev.mac_evals, ev.list_pushes) == (ev_o["interactions"], ev_o["mac_evals"],
                                                               ev_o["list_pushes"])
    sel = np.arange(len(mass)) if targets is None else np.asarray(targets)
    err = g2.force_error(s.acc[sel], acc_o[sel])
    assert err["median"] <= MED_TOL and err["p99"] <= P99_TOL, err
    if pot:
        rel = np.abs(pot_g[sel] - pot_o[sel]) / np.abs(pot_o[sel])
        assert np.median(rel) <= MED_TOL and np.quantile(rel, 0.99) <= P99_TOL
    return s, ev, err


def test_walk_fp32_range_guards(g2, oracle):
    """ADVICE r1 (walk.cu guard): a tiny but FP32-normal softening with unit masses makes the self
    pair's factor m / eps^3 overflow FP32 (1e42); the guarded flush drops the exact zero separation
    (traversal.cpp:73) and the forces stay finite and within the FP32 bar.  A total mass x G beyond
    the FP32 range is rejected as a data error instead of producing inf list entries."""
    mass, pos, _ = plummer(4096, seed=5)
    mass = np.ones_like(mass)
    am = np.full(len(mass), 4096.0)
    s, _, _ = walk_case(g2, oracle, mass, pos, am, g2.GravParams(1.0, 1e-14, 2.0 ** -9))
    assert np.isfinite(s.acc).all()
    big = np.full(len(mass), 1e36)
    with pytest.raises(g2.DataError):
        eng = g2.GravityEngine(g2.GravParams(1.0, 2.0 ** -5, 2.0 ** -9))
        eng.build(g2.ParticleSystem(big, pos))


@pytest.mark.parametrize("dacc", [2.0 ** -1, 2.0 ** -3, 2.0 ** -9, 2.0 ** -15])
def test_walk_plummer_dacc(g2, oracle, dacc):
    mass, pos, _ = plummer(32768, seed=2)
    am = np.full(len(mass), 1.0)
    walk_case(g2, oracle, mass, pos, am, g2.GravParams(1.0, 2.0 ** -5, dacc))


def test_walk_golden_m31(g2):
    g = load_golden("m31_16384")
    s = g2.ParticleSystem(g["mass"], g["pos"], acc_old_mag=g["acc_old_mag"])
    eng = g2.GravityEngine(g2.GravParams(1.0, 2.0 ** -5, 2.0 ** -9))
    eng.build(s)
    ev = eng.evaluate(s)
    assert [ev.interactions, ev.mac_evals, ev.list_pushes] == list(g["events"])
    err = g2.force_error(s.acc, g["acc"])
    assert err["median"] <= MED_TOL and err["p99"] <= P99_TOL, err


@pytest.mark.parametrize("gs", [1, 7, 16, 31])
def test_walk_group_sizes(g2, oracle, gs):
    mass, pos, _ = plummer(8192, seed=gs)
    am = np.random.default_rng(gs).uniform(0.5, 2.0, len(mass))
    walk_case(g2, oracle, mass, pos, am, g2.GravParams(1.0, 2.0 ** -5, 2.0 ** -6), g2.EngineConfig(group_size=gs))


def test_walk_potential_and_targets(g2, oracle):
    mass, pos, _ = plummer(16384, seed=9)
    am = np.full(len(mass), 0.7)
    rng = np.random.default_rng(4)
    targets = rng.choice(len(mass), 3000, replace=False).astype(np.uint32)
    walk_case(g2, oracle, mass, pos, am, g2.GravParams(1.0, 2.0 ** -5, 2.0 ** -9), targets=targets, pot=True)


def test_walk_zero_softening_and_geometric(g2, oracle):
    mass, pos, _ = random_cloud(5000, 7)
    # a_min == 0 everywhere selects the geometric MAC (engine.cpp:66)
    walk_case(g2, oracle, mass, pos, np.zeros(5000), g2.GravParams(1.0, 0.0, 2.0 ** -9))
    walk_case(g2, oracle, mass, pos, np.full(5000, 2.0), g2.GravParams(1.0, 0.0, 2.0 ** -9))


def test_two_body_leaf_path(g2, oracle):
    # test_gravity.cpp:187-200: a two-body walk is the leaf path == direct sum (FP32 here)
    mass = np.array([1.5, 0.5])
    pos = np.array([[-0.4, 0.1, 0.0], [0.6, -0.2, 0.3]])
    p = g2.GravParams(1.0, 0.05, 0.5)
    s = g2.ParticleSystem(mass, pos, acc_old_mag=np.ones(2))
    eng = g2.GravityEngine(p)
    eng.build(s)
    eng.evaluate(s)
    ref = oracle.direct_sum(mass, pos, eps=0.05)
    assert np.allclose(s.acc, ref, rtol=1e-6, atol=0)


def test_frontier_cap_resource_error(g2):
    mass, pos, _ = plummer(512, seed=3)  # test_gravity.cpp:261-272
    s = g2.ParticleSystem(mass, pos, acc_old_mag=np.ones(512))
    eng = g2.GravityEngine(g2.GravParams(1.0, 0.02, 2.0 ** -12), g2.EngineConfig(frontier_cap=2))
    eng.build(s)
    with pytest.raises(g2.ResourceError):
        eng.evaluate(s)


def test_list_capacity_and_errors(g2):
    mass, pos, _ = plummer(1024, seed=8)
    res = []
    for cap in (32, 64, 256, 1024):  # results independent of capacity (test_gravity.cpp:213-229)
        s = g2.ParticleSystem(mass, pos, acc_old_mag=np.ones(1024))
        eng = g2.GravityEngine(g2.GravParams(1.0, 0.02, 2.0 ** -6), g2.EngineConfig(list_capacity=cap))
        eng.build(s)
        res.append(eng.evaluate(s))
    assert all(r == res[0] for r in res)
    with pytest.raises(g2.DataError):
        g2.GravityEngine(g2.GravParams(), g2.EngineConfig(group_size=0))
    with pytest.raises(g2.DataError):
        g2.GravityEngine(g2.GravParams(dacc=0.0))
    with pytest.raises(g2.DataError):
        g2.GravityEngine().evaluate(g2.ParticleSystem(mass, pos))  # no tree


# ---------------------------------------------------------------- bootstrap, direct sum, integrator
def test_direct_sum_bitexact(g2, oracle):
    mass, pos, _ = plummer(3000, seed=12)
    for eps in (0.0, 2.0 ** -5):
        a = g2.direct_sum(g2.ParticleSystem(mass, pos), g2.GravParams(1.0, eps))
        assert np.array_equal(a, oracle.direct_sum(mass, pos, eps=eps))
    pos[5] = pos[6]
    with pytest.raises(g2.SingularityError):
        g2.direct_sum(g2.ParticleSystem(mass, pos), g2.GravParams(1.0, 0.0))


def test_bootstrap_direct_golden(g2):
    g = load_golden("plummer_4096")
    s = g2.ParticleSystem(g["mass"], g["pos"])
    ev = g2.GravityEngine(g2.GravParams(1.0, 2.0 ** -5, 2.0 ** -9)).bootstrap(s)
    assert ev.interactions == 4096 * 4095
    assert np.array_equal(s.acc, g["boot_acc"])
    assert np.array_equal(s.acc_old_mag, g["acc_old_mag"])


def test_predict_and_block_level_bitexact(g2, oracle):
    rng = np.random.default_rng(5)
    n = 10000
    s = g2.ParticleSystem(np.ones(n), rng.normal(size=(n, 3)), rng.normal(size=(n, 3)), rng.normal(size=(n, 3)))
    po, vo = oracle.predict(s.pos, s.vel, s.acc, 0.0123)
    g2.predict(s, 0.0123)
    assert np.array_equal(s.pos, po) and np.array_equal(s.vel, vo)
    amag = np.concatenate([[0.0, 1e-300, 1e300], 10.0 ** rng.uniform(-6, 6, 5000)])
    sch = g2.StepScheme(eta=0.5, dt_max=1 / 16)
    lv = g2.block_level(amag, sch, 2.0 ** -5)
    assert np.array_equal(lv, [oracle.block_level(a, 0.5, 1 / 16, True, 0, 2.0 ** -5) for a in amag])


def test_simulation_step_parity(g2, ref):
    """Simulation.step vs the reference Simulation from identical inputs (per-step, tolerance)."""
    m, p, v = ref.sample_model("plummer", 4096, 3)
    rs = ref.simulation(m, p, v, eps=2.0 ** -5, dt_max=1 / 64, threads=4)
    rs.init()
    rs.set_fixed_rebuild_interval(4)
    gs = g2.Simulation(g2.ParticleSystem(m, p, v), g2.GravParams(1.0, 2.0 ** -5, 2.0 ** -9),
                       g2.StepScheme(dt_max=1 / 64))
    gs.init()
    gs.set_fixed_rebuild_interval(4)
    r0, g0 = rs.state(), gs.system()
    assert np.array_equal(g0.acc, r0["acc"])  # direct bootstrap is bit-exact
    assert np.array_equal(g0.level, r0["level"])
    for _ in range(6):
        a, b = rs.step(), gs.step()
        assert a["active"] == b.active and a["rebuilt"] == b.rebuilt
    r1, g1 = rs.state(), gs.system()
    assert g1.time == r1["time"]
    # FP32 forces (median <= 1e-5, p99 <= 1e-4 relative) integrated over 6 steps of dt = 1/64:
    # the bulk agrees to ~1e-10; the worst particle (closest pair) within 1e-7
    dpos, dvel = np.abs(g1.pos - r1["pos"]), np.abs(g1.vel - r1["vel"])
    assert np.median(dpos) < 1e-9 and np.max(dpos) < 1e-7
    assert np.median(dvel) < 1e-7 and np.max(dvel) < 1e-5


def test_direct_sum_targets(g2, oracle):
    from paper_1811_02761_b200.gravitree import direct_sum_targets
    mass, pos, _ = plummer(40000, seed=21)
    tg = np.random.default_rng(1).choice(len(mass), 500, replace=False)
    a = direct_sum_targets(g2.ParticleSystem(mass, pos), tg, g2.GravParams(1.0, 2.0 ** -5))
    ref = oracle.direct_sum(mass, pos, eps=2.0 ** -5)[tg]
    rel = np.linalg.norm(a - ref, axis=1) / np.linalg.norm(ref, axis=1)
    assert rel.max() < 1e-12


def test_config1_plummer_2e16_full_step(g2, ref):
    """BASELINE config 1: Plummer 2^16, one full step (build_structure + refresh + evaluate(all))
    on the bootstrapped state, against the reference library on the same input."""
    m, p, _ = ref.sample_model("plummer", 1 << 16, 1)
    e = ref.engine(eps=2.0 ** -5, dacc=2.0 ** -9, threads=0)
    _, amag, _ = e.bootstrap(m, p)  # direct summation (n <= 65536), FP64
    e.build(m, p)
    acc_r, _, ev_r = e.evaluate(m, p, amag)
    s = g2.ParticleSystem(m, p)
    eng = g2.GravityEngine(g2.GravParams(1.0, 2.0 ** -5, 2.0 ** -9))
    eng.bootstrap(s)
    assert np.array_equal(s.acc_old_mag, amag)  # bit-exact bootstrap
    eng.build_structure(s)
    eng.refresh(s)
    ev = eng.evaluate(s)
    assert (ev.interactions, ev.mac_evals, ev.list_pushes) == (ev_r["interactions"], ev_r["mac_evals"],
                                                               ev_r["list_pushes"])
    err = g2.force_error(s.acc, acc_r)
    assert err["median"] <= MED_TOL and err["p99"] <= P99_TOL, err


@pytest.mark.slow
def test_full_size_tree_bitexact_m31_2e23(g2, ref):
    """BASELINE config 3 input at full size: the bench's M31 N=2^23 tree (keys, perm, cells,
    nodes) equals the reference build_tree bit for bit."""
    from paper_1811_02761_b200.gravitree import sample_model
    m, p, _ = sample_model("m31", 1 << 23, 1)
    t = gpu_tree(g2, m, p)
    rt = ref.build_tree(m, p)
    for k in ("bbox", "keys", "perm", "rank", "cells", "depth", "nodes"):
        assert np.array_equal(getattr(t, k), getattr(rt, k)), k


@pytest.mark.parametrize("cluster", [10, 100])
def test_simulation_rebuild_ties(g2, oracle, cluster):
    """Simulation rebuilds sort keys in storage order and repair equal-key runs to the reference's
    (key, original index) order in place (runs <= 64) or by the id-order sort (longer runs):
    engine().tree() after a step equals build_tree on the step's positions, bit for bit."""
    mass, pos, vel = plummer(20000, seed=5)
    rng = np.random.default_rng(cluster)
    at = rng.choice(len(mass), cluster, replace=False)
    pos[at] = pos[at[0]]  # a run of identical positions (identical keys), scattered ids
    vel[at] = vel[at[0]]
    sim = g2.Simulation(g2.ParticleSystem(mass, pos, vel), g2.GravParams(1.0, 2.0 ** -5, 2.0 ** -9),
                        g2.StepScheme(dt_max=1 / 64))
    sim.init()
    sim.set_rebuild_every_step(True)
    for _ in range(2):
        sim.step()
        t, st = sim.tree(), sim.system()
        ref = oracle.build_tree(mass, st.pos)
        for k in ("keys", "perm", "rank", "cells", "depth"):
            assert np.array_equal(getattr(t, k), getattr(ref, k)), k


@pytest.mark.parametrize("cluster", [0, 40, 5000, 9000])
def test_simulation_rebuild_bucket_sort(g2, oracle, cluster):
    """Rebuild sorts of n >= 2^15 go through the bucket sort of the nearly sorted storage order
    (bucket_sort.cu): after every rebuilding step the tree equals build_tree on the step's positions
    bit for bit.  cluster > 0 puts that many particles on one position: 40 exercises the in-place tie
    repair inside one bucket; 5000 fills a bucket beyond the small local sort (4096 keys), so the
    1024-thread instance sorts it (and the over-long tie run then takes the id-order sort); 9000
    overflows a bucket region (8192): the sort's gate opens and the id-order sort redoes the build."""
    mass, pos, vel = plummer(1 << 17, seed=7)
    if cluster:
        at = np.random.default_rng(cluster).choice(len(mass), cluster, replace=False)
        pos[at] = pos[at[0]]
        vel[at] = 0.0
    sim = g2.Simulation(g2.ParticleSystem(mass, pos, vel), g2.GravParams(1.0, 2.0 ** -5, 2.0 ** -9),
                        g2.StepScheme(dt_max=1 / 64))
    sim.init()
    sim.set_rebuild_every_step(True)
    for _ in range(3):
        sim.step()
        t, st = sim.tree(), sim.system()
        ref = oracle.build_tree(mass, st.pos)
        for k in ("bbox", "keys", "perm", "rank", "cells", "depth"):
            assert np.array_equal(getattr(t, k), getattr(ref, k)), k
    sorts, fallbacks = sim.sort_stats()
    assert sorts + fallbacks == 4  # init + 3 steps
    if cluster == 9000:
        assert fallbacks == 4
    else:
        assert sorts >= 3  # the steps' rebuilds (the init build's storage order is the sampler's)


@pytest.mark.slow
def test_config2_plummer_2e20_block_steps(g2, ref):
    """BASELINE config 2: Plummer 2^20, 16 block time steps of the GPU Simulation (reference driver
    defaults, fixed rebuild interval 8); at each rebuild the tree equals the reference build_tree of
    that step's positions bit for bit, and after 16 steps a fresh reference walk of the evolved state
    (sampled sinks) matches the GPU walk within the FP32 tolerance, events exact."""
    m, p, v = ref.sample_model("plummer", 1 << 20, 1)
    params = g2.GravParams(1.0, 2.0 ** -5, 2.0 ** -9)
    sim = g2.Simulation(g2.ParticleSystem(m, p, v), params, g2.StepScheme())
    sim.init()  # n > 65536: builds the tree and bootstraps with the geometric walk (engine.cpp:95-100)
    sim.set_fixed_rebuild_interval(8)
    t, rt = sim.tree(), ref.build_tree(m, p)
    for k in ("bbox", "keys", "perm", "rank", "cells", "depth"):
        assert np.array_equal(getattr(t, k), getattr(rt, k)), k
    rebuilds = 0
    for _ in range(16):
        r = sim.step()
        if r.rebuilt:
            rebuilds += 1
            st = sim.system()
            t, rt = sim.tree(), ref.build_tree(m, st.pos)
            for k in ("bbox", "keys", "perm", "rank", "cells", "depth"):
                assert np.array_equal(getattr(t, k), getattr(rt, k)), k
    assert rebuilds >= 1
    st = sim.system()
    tg = np.sort(np.random.default_rng(5).choice(len(m), 8192, replace=False)).astype(np.uint32)
    e = ref.engine(eps=params.eps, dacc=params.dacc, threads=0)
    e.build(m, st.pos)
    acc_r, _, ev_r = e.evaluate(m, st.pos, st.acc_old_mag, targets=tg)
    s = g2.ParticleSystem(m, st.pos, acc_old_mag=st.acc_old_mag)
    eng = g2.GravityEngine(params)
    eng.build(s)
    ev = eng.evaluate(s, targets=tg)
    assert (ev.interactions, ev.mac_evals, ev.list_pushes) == (ev_r["interactions"], ev_r["mac_evals"],
                                                               ev_r["list_pushes"])
    err = g2.force_error(s.acc[tg], acc_r[tg])
    assert err["median"] <= MED_TOL and err["p99"] <= P99_TOL, err


@pytest.mark.parametrize("leaf_cap,group_size", [(1, 32), (16, 7), (3, 32)])
def test_simulation_configs_tree_and_forces(g2, ref, leaf_cap, group_size):
    """Non-default EngineConfig through the Simulation path (storage-order rebuild sort, tie repair,
    non-recursive split, bottom-up calcNode, walk): after each rebuilding step the tree equals the
    reference build_tree of that step's positions, and a fresh walk of the evolved state matches the
    reference (events exact, FP32 tolerance)."""
    m, p, v = ref.sample_model("m31", 40000, 2)
    params = g2.GravParams(1.0, 2.0 ** -5, 2.0 ** -9)
    cfg = g2.EngineConfig(leaf_cap=leaf_cap, group_size=group_size)
    sim = g2.Simulation(g2.ParticleSystem(m, p, v), params, g2.StepScheme(dt_max=1 / 16), cfg)
    sim.init()
    sim.set_rebuild_every_step(True)
    for _ in range(3):
        sim.step()
        st, t = sim.system(), sim.tree()
        rt = ref.build_tree(m, st.pos, leaf_cap=leaf_cap)
        for k in ("keys", "perm", "rank", "cells", "depth"):
            assert np.array_equal(getattr(t, k), getattr(rt, k)), k
    st = sim.system()
    e = ref.engine(eps=params.eps, dacc=params.dacc, leaf_cap=leaf_cap, group_size=group_size, threads=0)
    e.build(m, st.pos)
    acc_r, _, ev_r = e.evaluate(m, st.pos, st.acc_old_mag)
    s = g2.ParticleSystem(m, st.pos, acc_old_mag=st.acc_old_mag)
    eng = g2.GravityEngine(params, cfg)
    eng.build(s)
    ev = eng.evaluate(s)
    assert (ev.interactions, ev.mac_evals, ev.list_pushes) == (ev_r["interactions"], ev_r["mac_evals"],
                                                               ev_r["list_pushes"])
    err = g2.force_error(s.acc, acc_r)
    assert err["median"] <= MED_TOL and err["p99"] <= P99_TOL, err
