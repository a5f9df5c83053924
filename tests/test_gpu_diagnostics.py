"""GPU: compute_diagnostics (diagnostics.cpp:10-38) against the reference library, and the
reference's energy-based integrator tests (test_dynamics.cpp:20-45, 141-158; test_models.cpp:90-94)
through the device-resident Simulation."""
import math

import numpy as np
import pytest

from conftest import plummer

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def g2():
    import paper_1811_02761_b200 as g2mod
    return g2mod


def rel(a, b):
    s = max(abs(a), abs(b))
    return abs(a - b) / s if s else 0.0


def moving_plummer(n, seed):
    mass, pos, _ = plummer(n, seed=seed)
    vel = np.random.default_rng(seed + 100).normal(scale=0.3, size=(n, 3))
    return mass, pos, vel


def test_diagnostics_direct_path(g2, ref):
    mass, pos, vel = moving_plummer(4096, 3)
    p = g2.GravParams(1.0, 2.0 ** -5, 2.0 ** -9)
    d = g2.compute_diagnostics(g2.ParticleSystem(mass, pos, vel), p)
    r = ref.diagnostics(mass, pos, vel, G=p.G, eps=p.eps, dacc=p.dacc, threads=4)
    assert rel(d.kinetic, r["kinetic"]) < 1e-13
    assert rel(d.potential, r["potential"]) < 1e-12  # FP64 pair sums, different summation order
    assert rel(d.total, r["total"]) < 1e-12
    assert rel(d.virial_ratio, r["virial_ratio"]) < 1e-12
    assert np.allclose(d.momentum, r["momentum"], rtol=0, atol=1e-13)


def test_diagnostics_tree_path(g2, ref):
    # beyond kDirectPotentialLimit = 2^17: the dacc = 2^-20 tree potential with the system's acc_old_mag
    mass, pos, vel = moving_plummer((1 << 17) + 4096, 5)
    am = np.random.default_rng(2).uniform(0.5, 2.0, len(mass))
    p = g2.GravParams(1.0, 2.0 ** -5, 2.0 ** -9)
    for amag in (None, am):  # zeros: geometric MAC (a fresh ParticleSystem), else the acceleration MAC
        s = g2.ParticleSystem(mass, pos, vel, acc_old_mag=amag)
        d = g2.compute_diagnostics(s, p)
        r = ref.diagnostics(mass, pos, vel, acc_old_mag=amag, G=p.G, eps=p.eps, dacc=p.dacc)
        assert rel(d.kinetic, r["kinetic"]) < 1e-13
        assert rel(d.potential, r["potential"]) < 1e-6  # FP32 tree potentials
        assert rel(d.virial_ratio, r["virial_ratio"]) < 1e-6


def test_diagnostics_singularity(g2):
    mass, pos, vel = moving_plummer(256, 1)
    pos[7] = pos[3]
    with pytest.raises(g2.SingularityError):
        g2.compute_diagnostics(g2.ParticleSystem(mass, pos, vel), g2.GravParams(1.0, 0.0, 2.0 ** -9))


def test_plummer_sample_near_virial_equilibrium(g2):
    # test_models.cpp:90-94 on the library's bit-identical sampler
    from paper_1811_02761_b200.gravitree import sample_model
    m, p, v = sample_model("plummer", 50000, 11)
    d = g2.compute_diagnostics(g2.ParticleSystem(m, p, v), g2.GravParams())
    assert abs(d.virial_ratio - 1.0) < 0.1


def eccentric_binary(a=1.0, e=0.5):
    # test_support.hpp:64-74
    r_apo = a * (1.0 + e)
    v_rel = math.sqrt((1.0 - e) / (a * (1.0 + e)))
    pos = np.array([[-0.5 * r_apo, 0.0, 0.0], [0.5 * r_apo, 0.0, 0.0]])
    vel = np.array([[0.0, -0.5 * v_rel, 0.0], [0.0, 0.5 * v_rel, 0.0]])
    return np.array([0.5, 0.5]), pos, vel


def kepler_energy_error(g2, dt, steps):
    # test_dynamics.cpp:20-36: max |dE/E| of an eccentric two-body orbit over one period at fixed dt
    mass, pos, vel = eccentric_binary()
    params = g2.GravParams(1.0, 0.0, 2.0 ** -20)
    sim = g2.Simulation(g2.ParticleSystem(mass, pos, vel), params,
                        g2.StepScheme(adaptive=False, fixed_level=0, dt_max=dt))
    sim.init()
    e0 = g2.compute_diagnostics(sim.system(), params).total
    worst = 0.0
    for _ in range(steps):
        sim.step()
        e = g2.compute_diagnostics(sim.system(), params).total
        worst = max(worst, abs((e - e0) / e0))
    return worst


def test_two_body_energy_converges_at_second_order(g2):
    # test_dynamics.cpp:141-158 (period 2 pi for a = 1, G M = 1)
    period = 2.0 * math.pi
    dts = [period / 250.0, period / 500.0, period / 1000.0]
    errs = [kepler_energy_error(g2, dt, int(period / dt)) for dt in dts]
    assert errs[0] / errs[1] == pytest.approx(4.0, rel=0.5)
    x, y = np.log(dts), np.log(errs)
    slope = np.polyfit(x, y, 1)[0]
    assert slope == pytest.approx(2.0, rel=0.15)
