"""CPU: the C-ABI library loads and exports every entry point include/g2/capi.h
declares; host-side logic (defaults, measurement convention, force_error)."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "g2", "capi.h")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(g2_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    import paper_1811_02761_b200.gravitree as gt
    lib = ctypes.CDLL(gt.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_library_is_sm100a_only():
    import subprocess
    import paper_1811_02761_b200.gravitree as gt
    out = subprocess.run(["cuobjdump", "--list-elf", gt.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out and "sm_90" not in out


def test_defaults_match_reference():
    import paper_1811_02761_b200 as g2
    from paper_1811_02761_b200.gravitree import _EngineConfig, _GravParams, _StepScheme, _TunerConfig, lib
    p, c, s, t = _GravParams(), _EngineConfig(), _StepScheme(), _TunerConfig()
    lib().g2_default_params(ctypes.byref(p))
    lib().g2_default_engine_config(ctypes.byref(c))
    lib().g2_default_step_scheme(ctypes.byref(s))
    lib().g2_default_tuner_config(ctypes.byref(t))
    assert (p.G, p.eps, p.dacc) == (1.0, 0.0, 2.0 ** -9)  # particle_system.hpp:53-57
    assert (c.leaf_cap, c.group_size, c.list_capacity, c.frontier_cap, c.count_ops, c.bootstrap_theta,
            c.bootstrap_direct_limit) == (8, 32, 1024, 0, 1, 0.5, 65536)  # engine.hpp:14-23
    assert (s.eta, s.dt_max, s.adaptive, s.fixed_level) == (0.5, 0.0625, 1, 0)  # integrator.hpp:18-23
    assert (t.min_interval, t.max_interval, t.initial_interval) == (1, 128, 8)  # rebuild_tuner.hpp:9-13
    d = g2.EngineConfig()
    assert (d.leaf_cap, d.group_size, d.list_capacity, d.bootstrap_direct_limit) == (8, 32, 1024, 65536)


def test_op_counter_convention():
    import paper_1811_02761_b200 as g2
    c = g2.count_walk_ops(g2.TraversalEvents(1, 1, 1))  # test_perflab.cpp:21-29
    assert (c["fp_fma"], c["fp_add"], c["fp_mul"], c["fp_rsqrt"], c["integer"]) == (9, 5, 5, 1, 16)
    assert g2.walk_flops(g2.TraversalEvents(1, 0, 0)) == 27.0
    assert g2.walk_flops(g2.TraversalEvents(0, 1, 0)) == 5.0
    with pytest.raises(g2.DataError):
        g2.flops_estimate(g2.TraversalEvents(1, 0, 0), 0.0)


def test_force_error_semantics():
    import paper_1811_02761_b200 as g2
    ref = np.array([[1.0, 0, 0], [0, 2.0, 0], [0, 0, 4.0]])  # test_gravity.cpp:274-300
    assert g2.force_error(ref, ref) == {"median": 0.0, "p99": 0.0, "max": 0.0, "excluded": 0}
    s = g2.force_error(1.01 * ref, ref)
    assert abs(s["median"] - 0.01) < 1e-12 and abs(s["max"] - 0.01) < 1e-12
    s = g2.force_error(np.array([[1.0, 0, 0], [5, 5, 5]]), np.array([[1.0, 0, 0], [0, 0, 0]]))
    assert s["excluded"] == 1 and s["max"] == 0.0


def test_no_gpu_calls_fail_loudly():
    """Without a device the library reports an error instead of computing on the CPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_1811_02761_b200 as g2
    with pytest.raises(g2.InternalError):
        g2.GravityEngine()


@pytest.mark.parametrize("model,n", [("m31", 20001), ("plummer", 3001), ("hernquist", 2048), ("nfw", 999),
                                     ("disk", 4097)])
def test_sampler_bit_identical_to_reference(ref, model, n):
    """The bench input generator (csrc/ics.cpp, multithreaded) reproduces the reference's
    sample_model (models.cpp:442-460) bit for bit."""
    from paper_1811_02761_b200.gravitree import sample_model
    a = ref.sample_model(model, n, 1)
    b = sample_model(model, n, 1, threads=4)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def test_product_autotune_matches_reference(ref):
    """g2_autotune (the Simulation's RebuildTuner logic in libg2, host code: callable without a GPU)
    against the reference library's autotune_rebuild (rebuild_tuner.cpp:28-61)."""
    import ctypes as C

    import numpy as np

    from paper_1811_02761_b200.gravitree import lib
    f = lib().g2_autotune
    f.restype = C.c_size_t
    rng = np.random.default_rng(11)
    hists = [[1.0] * 8, [1.0 + k for k in range(16)], [5.0], list(rng.uniform(0, 3, 11)),
             list(np.cumsum(rng.uniform(0, 0.2, 40)) + 1.0), [2.0] * 8]
    for hist in hists:
        h = np.ascontiguousarray(hist, dtype=np.float64)
        for bt in (0.0, 1e-4, 10.0, 1e6):
            for lo, hi, cur in ((1, 128, 8), (1, 32, 8), (2, 64, 13)):
                got = f(C.c_double(bt), C.c_size_t(len(h)), h.ctypes.data_as(C.c_void_p), C.c_size_t(lo),
                        C.c_size_t(hi), C.c_size_t(cur))
                assert got == ref.autotune(bt, hist, lo, hi, cur), (hist, bt, lo, hi, cur)
