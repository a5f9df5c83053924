"""The committed bench line (profiles/r2_bench_line.json, produced by `python bench.py` on a B200)
carries every key of the bench contract, and the reference arm's line its own."""
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def load(name):
    with open(os.path.join(ROOT, "profiles", name)) as f:
        return json.load(f)


def test_bench_line_contract():
    d = load("r2_bench_line.json")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["warmup"] >= 3 and d["higher_is_better"] is False and d["unit"] == "s/step"
    assert abs(d["ms_per_step"] - 1e3 * d["value"]) < 1e-9 * max(1.0, d["ms_per_step"])
    assert "workload" in d["config"] and "l2" in d["config"]
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r, k
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    c = d["cpu_baseline"]
    for k in ("value", "unit", "cores", "kind", "sample"):
        assert k in c, k
    assert c["kind"] in ("reference", "port") and c["cores"] >= 1
    e = d["e2e"]
    for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert k in e, k
    assert e["value"] > d["value"] and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    assert not set(d["clocks"]["reasons"]) & {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}


def test_reference_arm_line_contract():
    d = load("r2_reference_arm.json")
    g = load("r2_bench_line.json")
    # the driver divides the arms only when metric, unit and config match
    assert d["metric"] == g["metric"] and d["unit"] == g["unit"] and d["config"] == g["config"]
    # measured, not extrapolated: the timed steps fit in the timed wall clock
    assert d["steps"] * d["value"] <= d["timed_wall_seconds"] * (1 + 1e-6)
    assert d["impl"] == "reference" and d["unit"] == "s/step" and d["higher_is_better"] is False
    assert d["cpu_baseline"]["value"] == d["value"] and d["e2e"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


def test_both_arms_share_metric_unit_config(ref):
    """The reference arm, run here on a small input, prints the SAME metric string, unit and config as
    the g2 arm would for the same arguments (the driver divides the two only when they match), and its
    value is a measured full step: steps x value fits inside the timed wall clock (no extrapolation)."""
    import subprocess
    import sys
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--n", "4096",
                          "--model", "plummer", "--steps", "2", "--warmup", "3"], capture_output=True, text=True,
                         timeout=600, check=True).stdout.strip().splitlines()[-1]
    d = json.loads(out)
    sys.path.insert(0, ROOT)
    import bench
    args = bench.parse_args_list(["--n", "4096", "--model", "plummer", "--steps", "2", "--warmup", "3"])
    assert d["metric"] == bench.metric_name(args)
    assert d["config"] == bench.workload_config(args)
    assert d["unit"] == "s/step" and d["higher_is_better"] is False
    assert d["steps"] * d["value"] <= d["timed_wall_seconds"] * (1 + 1e-6)
    assert d["events_last_step"]["interactions"] > 0
