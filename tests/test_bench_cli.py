"""The reference CLI's benchmark drivers (tools/main.cpp:187-272) on the device: predict_speedup
fixed points (test_perflab.cpp:48-85) on CPU, and `tools/bench_cli.py accuracy|scaling` on a B200
with the reference's CSV schemas."""
import csv
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ops(integer=0, fma=0, add=0, mul=0):
    return dict(integer=integer, fp_fma=fma, fp_add=add, fp_mul=mul, fp_rsqrt=0)


def test_predict_speedup_fixed_points():
    import numpy as np

    from paper_1811_02761_b200.gravitree import DataError, predict_speedup
    assert predict_speedup(_ops(add=10)) == pytest.approx(1.5, rel=1e-15)
    assert predict_speedup(_ops(integer=10, add=10)) == pytest.approx(3.0, rel=1e-15)
    assert predict_speedup(_ops(integer=4_670_000_000, fma=10_000_000_000)) == pytest.approx(2.2005, rel=1e-4)
    with pytest.raises(DataError):
        predict_speedup(_ops())
    rng = np.random.default_rng(5)
    for _ in range(200):
        i, f, a, m = (int(x) for x in rng.integers(0, 10000, 4))
        s = predict_speedup(_ops(i, f + 1, a, m))
        assert 1.5 - 1e-12 <= s <= 3.0 + 1e-12
        assert predict_speedup(_ops(7 * i, 7 * (f + 1), 7 * a, 7 * m)) == pytest.approx(s, rel=1e-12)


def _run(args, tmp_path):
    out = str(tmp_path / "o.csv")
    subprocess.run([sys.executable, os.path.join(ROOT, "tools", "bench_cli.py")] + args + ["--out", out],
                   check=True, cwd=ROOT, timeout=600)
    with open(out) as f:
        return list(csv.reader(f))


@pytest.mark.gpu
def test_bench_accuracy_csv(tmp_path):
    rows = _run(["accuracy", "--dacc", "2^-3", "2^-9", "2^-15", "--steps", "2"], tmp_path)
    assert rows[0] == ["dacc", "t_step", "t_walk", "t_node", "t_build", "err_median", "err_p99",
                       "interactions_per_particle", "int_ops", "fp_ops", "predicted_speedup"]
    body = [[float(x) for x in r] for r in rows[1:]]
    assert [r[0] for r in body] == [2.0 ** -3, 2.0 ** -9, 2.0 ** -15]
    assert all(r[1] > 0 and r[2] > 0 for r in body)
    err = [r[5] for r in body]
    assert err[0] > err[1] > err[2] and err[2] < 1e-4  # tighter dacc, smaller error
    ipp = [r[7] for r in body]
    assert ipp[0] < ipp[1] < ipp[2] <= 4096
    assert all(1.5 <= r[10] <= 3.0 for r in body)
    assert all(rows[i][8].isdigit() and rows[i][9].isdigit() for i in range(1, 4))


@pytest.mark.gpu
def test_bench_scaling_csv(tmp_path):
    rows = _run(["scaling", "--n", "16384", "65536", "--steps", "2"], tmp_path)
    assert rows[0] == ["n", "t_step", "t_walk", "t_node", "t_build", "t_predict", "t_correct"]
    assert [r[0] for r in rows[1:]] == ["16384", "65536"]
    assert all(float(x) >= 0 for r in rows[1:] for x in r[1:])
