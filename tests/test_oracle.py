"""CPU: pin the C restatement (oracle/g2_oracle.c) before trusting it as the
GPU checker — against the golden fixtures (reference outputs, always
available) and, where oracle/_ref was built, against the reference library
itself on fresh inputs.  Closed forms follow the reference's own tests."""
import numpy as np
import pytest

from conftest import load_golden, plummer, random_cloud


@pytest.mark.parametrize("name", ["plummer_4096", "m31_16384"])
def test_oracle_matches_golden(oracle, name):
    g = load_golden(name)
    t = oracle.build_tree(g["mass"], g["pos"])
    for k in ("bbox", "keys", "perm", "rank", "cells", "depth", "nodes"):
        assert np.array_equal(getattr(t, k), g["tree_" + k]), k
    boot = oracle.direct_sum(g["mass"], g["pos"], eps=2.0 ** -5)
    assert np.array_equal(boot, g["boot_acc"])
    assert np.array_equal(np.sqrt((boot * boot).sum(1)), g["acc_old_mag"]) or np.allclose(
        np.sqrt((boot * boot).sum(1)), g["acc_old_mag"], rtol=1e-15, atol=0)
    acc, _, ev = oracle.evaluate(g["mass"], g["pos"], g["acc_old_mag"], eps=2.0 ** -5, dacc=2.0 ** -9)
    assert [ev["interactions"], ev["mac_evals"], ev["list_pushes"]] == list(g["events"])
    assert np.array_equal(acc, g["acc"])


@pytest.mark.parametrize("model,n", [("plummer", 3000), ("m31", 5000), ("hernquist", 2000), ("disk", 2000)])
def test_oracle_matches_reference(oracle, ref, model, n):
    mass, pos, _ = ref.sample_model(model, n, 7)
    t, rt = oracle.build_tree(mass, pos), ref.build_tree(mass, pos)
    for k in ("bbox", "keys", "perm", "rank", "cells", "depth", "nodes"):
        assert np.array_equal(getattr(t, k), getattr(rt, k)), k
    e = ref.engine(eps=0.01, dacc=2.0 ** -6, group_size=17, threads=2)
    e.build(mass, pos)
    am = np.random.default_rng(1).uniform(0.1, 3.0, n)
    targets = np.random.default_rng(2).choice(n, n // 3, replace=False).astype(np.uint32)
    a1, p1, ev1 = e.evaluate(mass, pos, am, targets=targets, with_potential=True)
    a2, p2, ev2 = oracle.evaluate(mass, pos, am, targets=targets, eps=0.01, dacc=2.0 ** -6, group_size=17,
                                  with_potential=True)
    assert ev1 == ev2
    assert np.array_equal(a1[targets], a2[targets]) and np.array_equal(p1[targets], p2[targets])
    g1 = ref.groups(pos, am, rt.rank, targets, 17)
    g2 = oracle.groups(pos, am, rt.rank, targets, 17)
    assert np.array_equal(g1, g2)


def test_oracle_integrator_matches_reference(oracle, ref):
    rng = np.random.default_rng(3)
    pos, vel, acc = rng.normal(size=(500, 3)), rng.normal(size=(500, 3)), rng.normal(size=(500, 3))
    a = oracle.predict(pos, vel, acc, 0.37)
    b = ref.predict(pos, vel, acc, 0.37)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    for amag in np.concatenate([[0.0, 1e-300, 1e300], 10.0 ** rng.uniform(-6, 6, 300)]):
        for eta, dtm in ((0.5, 1 / 16), (0.3, 1.0)):
            assert oracle.block_level(amag, eta, dtm, True, 0, 2.0 ** -5) == ref.block_level(amag, eta, dtm, True, 0,
                                                                                               2.0 ** -5)
    for hist in ([1.0] * 8, [1.0 + k for k in range(16)], [5.0], list(rng.uniform(0, 3, 11))):
        for bt in (0.0, 10.0, 1e6):
            assert oracle.autotune(bt, hist) == ref.autotune(bt, hist)


def test_oracle_closed_forms(oracle):
    # morton corners (test_tree.cpp:42-46) via a two-particle cube [-0.5, 0.5]^3
    t = oracle.build_tree(np.ones(2), np.array([[-0.5, -0.5, -0.5], [0.5, 0.5, 0.5]]))
    assert int(t.keys[0]) == 0 and int(t.keys[1]) == 0x7fffffffffffffff
    # single particle, 8 octants with leaf_cap 1 (test_tree.cpp:73-103)
    t = oracle.build_tree(np.array([2.0]), np.array([[0.3, -0.1, 0.7]]))
    assert len(t.cells) == 1 and t.nodes[0, 0] == 2.0 and t.nodes[0, 4] == 0.0
    pos = np.array([[sx, sy, sz] for sx in (-.25, .25) for sy in (-.25, .25) for sz in (-.25, .25)])
    t = oracle.build_tree(np.ones(8), pos, leaf_cap=1)
    assert len(t.cells) == 9 and t.cells[0, 1] == 8
    # direct sum: unit separation (test_gravity.cpp:30-37) and Newton III
    a = oracle.direct_sum(np.ones(2), np.array([[0.0, 0, 0], [1.0, 0, 0]]))
    assert a[0, 0] == 1.0 and a[1, 0] == -1.0
    # autotuner closed forms (test_dynamics.cpp:270-320)
    assert oracle.autotune(0.0, [2.0] * 8) == 128
    assert oracle.autotune(10.0, [1.0 + k for k in range(16)]) in (4, 5)
    assert oracle.autotune(1.0, [5.0], cur=13) == 13


def test_oracle_frontier_cap(oracle):
    mass, pos, _ = plummer(512, seed=3)
    from oracle.refpy import RefError
    with pytest.raises(RefError) as e:
        oracle.evaluate(mass, pos, np.ones(512), eps=0.02, dacc=2.0 ** -12, frontier_cap=2)
    assert e.value.code == 4


def test_oracle_force_accuracy_trend(oracle):
    """Median error vs direct summation falls with dacc (test_gravity.cpp:242-259)."""
    mass, pos, _ = random_cloud(2048, 5)
    ref = oracle.direct_sum(mass, pos, eps=0.02)
    from oracle.refpy import force_error
    meds = []
    for dacc in (2.0 ** -1, 2.0 ** -6, 2.0 ** -12):
        acc, _, _ = oracle.evaluate(mass, pos, np.ones(2048), eps=0.02, dacc=dacc)
        meds.append(force_error(acc, ref)["median"])
    assert meds[2] < meds[0]
