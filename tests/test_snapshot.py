"""OCTF snapshot I/O (snapshot.hpp:10-30, snapshot.cpp:65-121) against the reference library: byte-
identical files both ways, the reference's error messages, and (GPU) a Simulation loaded straight
from a snapshot equals one built from the same arrays."""
import os

import numpy as np
import pytest

from conftest import plummer


@pytest.fixture(scope="module")
def g2():
    import paper_1811_02761_b200 as g2mod
    return g2mod


def system(g2, n=1000, seed=4):
    mass, pos, _ = plummer(n, seed=seed)
    vel = np.random.default_rng(seed).normal(size=(n, 3))
    s = g2.ParticleSystem(mass, pos, vel)
    s.time = 0.375
    return s


def test_roundtrip_byte_identical_with_reference(g2, ref, tmp_path):
    s = system(g2)
    p = g2.GravParams(1.0, 2.0 ** -5, 2.0 ** -9)
    a, b = tmp_path / "g2.octf", tmp_path / "ref.octf"
    g2.write_snapshot(a, s, p)
    ref.write_snapshot(b, s.mass, s.pos, s.vel, s.time, p.G, p.eps)
    assert a.read_bytes() == b.read_bytes()
    assert not os.path.exists(str(a) + ".tmp")
    snap = g2.read_snapshot(b)
    assert snap.G == p.G and snap.eps == p.eps and snap.system.time == s.time
    for k in ("mass", "pos", "vel"):
        assert np.array_equal(getattr(snap.system, k), getattr(s, k))
    m, q, v, t, G, eps = ref.read_snapshot(a)
    assert np.array_equal(m, s.mass) and np.array_equal(q, s.pos) and np.array_equal(v, s.vel)
    assert (t, G, eps) == (s.time, p.G, p.eps)


@pytest.mark.parametrize("cut", [0, 2, 6, 12, 20, 28, 36, 40 + 8 * 10, 40 + 8 * 50 + 3, 40 + 8 * 200 - 1])
def test_truncation_messages_match_reference(g2, ref, tmp_path, cut):
    from oracle.refpy import RefError
    s = system(g2, n=50)
    full = tmp_path / "full.octf"
    g2.write_snapshot(full, s)
    bad = tmp_path / "cut.octf"
    bad.write_bytes(full.read_bytes()[:cut])
    with pytest.raises(RefError) as er:
        ref.read_snapshot(bad)
    with pytest.raises(g2.DataError) as eg:
        g2.read_snapshot(bad)
    assert str(eg.value) == er.value.msg


def test_header_errors_match_reference(g2, ref, tmp_path):
    from oracle.refpy import RefError
    s = system(g2, n=10)
    full = tmp_path / "ok.octf"
    g2.write_snapshot(full, s)
    data = bytearray(full.read_bytes())
    cases = {"magic": (2, ord("X")), "version": (4, 2)}
    for name, (at, val) in cases.items():
        d = bytearray(data)
        d[at] = val
        f = tmp_path / f"{name}.octf"
        f.write_bytes(bytes(d))
        with pytest.raises(RefError) as er:
            ref.read_snapshot(f)
        with pytest.raises(g2.DataError) as eg:
            g2.read_snapshot(f)
        assert str(eg.value) == er.value.msg
    d = bytearray(data)
    d[8:16] = bytes(8)  # n = 0
    f = tmp_path / "zero.octf"
    f.write_bytes(bytes(d))
    with pytest.raises(g2.DataError, match="zero particle count at byte 8"):
        g2.read_snapshot(f)
    with pytest.raises(g2.DataError, match="cannot open"):
        g2.read_snapshot(tmp_path / "missing.octf")


@pytest.mark.parametrize("n", [2 ** 61 + 1, 2 ** 64 - 1, 2 ** 40, 51])
def test_untrusted_particle_count(g2, ref, tmp_path, n):
    """A crafted header count must fail cleanly before anything is sized by it: 40 + 56 n wraps
    size_t for n = 2^61 + 1; otherwise the file is simply too short (the reference's truncation
    message, same byte offset, when the reference can allocate n particles)."""
    from oracle.refpy import RefError
    s = system(g2, n=50)
    full = tmp_path / "full.octf"
    g2.write_snapshot(full, s)
    d = bytearray(full.read_bytes())
    d[8:16] = n.to_bytes(8, "little")
    f = tmp_path / "crafted.octf"
    f.write_bytes(bytes(d))
    with pytest.raises(g2.DataError) as eg:
        g2.read_snapshot(f)
    if n == 51:
        with pytest.raises(RefError) as er:
            ref.read_snapshot(f)
        assert str(eg.value) == er.value.msg
    if n > (2 ** 64 - 1 - 40) // 56:
        assert "too large" in str(eg.value)
    else:
        assert "truncated" in str(eg.value)


@pytest.mark.gpu
def test_simulation_from_snapshot_untrusted_count(g2, tmp_path):
    s = system(g2, n=50)
    full = tmp_path / "full.octf"
    g2.write_snapshot(full, s)
    d = bytearray(full.read_bytes())
    d[8:16] = (2 ** 61 + 1).to_bytes(8, "little")
    f = tmp_path / "crafted.octf"
    f.write_bytes(bytes(d))
    with pytest.raises(g2.DataError, match="too large"):
        g2.Simulation.from_snapshot(f, dacc=2.0 ** -9)


@pytest.mark.gpu
def test_simulation_from_snapshot(g2, tmp_path):
    mass, pos, _ = plummer(20000, seed=8)
    vel = np.random.default_rng(8).normal(scale=0.2, size=(len(mass), 3))
    s = g2.ParticleSystem(mass, pos, vel)
    p = g2.GravParams(1.0, 2.0 ** -5, 2.0 ** -9)
    f = tmp_path / "ic.octf"
    g2.write_snapshot(f, s, p)
    a = g2.Simulation.from_snapshot(f, dacc=p.dacc, scheme=g2.StepScheme(dt_max=1 / 64))
    b = g2.Simulation(s, p, g2.StepScheme(dt_max=1 / 64))
    for sim in (a, b):
        sim.init()  # direct-sum bootstrap (n <= 65536): FP64, deterministic
    sa, sb = a.system(), b.system()
    for k in ("pos", "vel", "acc", "acc_old_mag", "level"):
        assert np.array_equal(getattr(sa, k), getattr(sb, k)), k
    for sim in (a, b):
        for _ in range(3):
            sim.step()
    # tree steps are deterministic (ordered combination of split groups): bit-identical runs
    sa, sb = a.system(), b.system()
    assert sa.time == sb.time
    assert np.array_equal(sa.pos, sb.pos) and np.array_equal(sa.vel, sb.vel)
    out = tmp_path / "out.octf"
    a.write_snapshot(out)
    back = g2.read_snapshot(out)
    assert np.array_equal(back.system.pos, sa.pos) and np.array_equal(back.system.mass, mass)
    assert back.system.time == sa.time and (back.G, back.eps) == (p.G, p.eps)
