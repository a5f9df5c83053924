"""GPU counterparts of the reference CLI's benchmark drivers (tools/main.cpp:187-272), same CSV
schemas and protocols, on the g2 Simulation / GravityEngine:

  python tools/bench_cli.py accuracy [--n 4096] [--model plummer] [--steps 8] [--dacc 2^-p ...] [--out accuracy.csv]
      per dacc (default grid 2^-1 .. 2^-20, main.cpp:35-39): Simulation(model, dacc) init + `steps` block
      steps (mean phase times; t_step = mean host wall time per step), then a full walk of the final
      state vs FP64 direct summation (force_error), interactions/particle and the op-count costing.
      predicted_speedup is the reference's overlap model with its default HardwareRatios (1.5).
  python tools/bench_cli.py scaling --n 65536 262144 ... [--steps 4] [--out scaling.csv]
      per N: mean phase times of `steps` block steps (main.cpp:238-272).
Numbers are written with %.17g like the reference's CsvBuilder (csv.cpp:32-36)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1811_02761_b200 as g2  # noqa: E402
from paper_1811_02761_b200.gravitree import sample_model  # noqa: E402


def fmt(v):
    return "%.17g" % v if isinstance(v, float) else str(v)


def write_csv(path, header, rows):
    with open(path + ".tmp", "w") as f:
        f.write(",".join(header) + "\n")
        for r in rows:
            f.write(",".join(fmt(x) for x in r) + "\n")
    os.replace(path + ".tmp", path)


def run_steps(sim, steps):
    sums = dict(walk_tree=0.0, calc_node=0.0, make_tree=0.0, predict=0.0, correct=0.0)
    wall = 0.0
    for _ in range(steps):
        r = sim.step()
        for k in sums:
            sums[k] += getattr(r.timings, k)
        wall += r.wall_seconds
    inv = 1.0 / steps if steps else 0.0
    return {k: v * inv for k, v in sums.items()}, wall * inv


def parse_dacc(s):
    return 2.0 ** -float(s[3:]) if s.startswith("2^-") else float(s)


def accuracy(a):
    grid = [parse_dacc(x) for x in a.dacc] if a.dacc else [2.0 ** -p for p in range(1, 21)]
    m, p, v = sample_model(a.model, a.n, a.seed)
    rows = []
    for dacc in grid:
        params = g2.GravParams(1.0, a.eps, dacc)
        sim = g2.Simulation(g2.ParticleSystem(m, p, v), params, g2.StepScheme())
        sim.init()
        t, wall = run_steps(sim, a.steps)
        probe = sim.system()
        eng = g2.GravityEngine(params)
        eng.build(probe)
        ev = eng.evaluate(probe)
        ref = g2.direct_sum(probe, params)
        err = g2.force_error(probe.acc, ref)
        ops = g2.count_walk_ops(ev)
        rows.append([dacc, wall, t["walk_tree"], t["calc_node"], t["make_tree"], err["median"], err["p99"],
                     ev.interactions / probe.n(), int(ops["integer"]),
                     int(ops["fp_fma"] + ops["fp_add"] + ops["fp_mul"]), g2.predict_speedup(ops)])
        print("dacc %.3e: err_median %.3e err_p99 %.3e" % (dacc, err["median"], err["p99"]), flush=True)
    write_csv(a.out, ["dacc", "t_step", "t_walk", "t_node", "t_build", "err_median", "err_p99",
                      "interactions_per_particle", "int_ops", "fp_ops", "predicted_speedup"], rows)


def scaling(a):
    rows = []
    for n in a.n:
        m, p, v = sample_model(a.model, n, a.seed)
        sim = g2.Simulation(g2.ParticleSystem(m, p, v), g2.GravParams(1.0, a.eps, parse_dacc(a.dacc_one)),
                            g2.StepScheme())
        sim.init()
        t, wall = run_steps(sim, a.steps)
        rows.append([int(n), wall, t["walk_tree"], t["calc_node"], t["make_tree"], t["predict"], t["correct"]])
        print("n %d: %.3e s/step (walk %.3e)" % (n, wall, t["walk_tree"]), flush=True)
    write_csv(a.out, ["n", "t_step", "t_walk", "t_node", "t_build", "t_predict", "t_correct"], rows)


def main():
    ap = argparse.ArgumentParser()
    sub = ap.add_subparsers(dest="cmd", required=True)
    pa = sub.add_parser("accuracy")
    pa.add_argument("--n", type=int, default=4096)
    pa.add_argument("--model", default="plummer")
    pa.add_argument("--seed", type=int, default=1)
    pa.add_argument("--dacc", nargs="*", default=[])
    pa.add_argument("--steps", type=int, default=8)
    pa.add_argument("--eps", type=float, default=0.03125)
    pa.add_argument("--out", default="accuracy.csv")
    ps = sub.add_parser("scaling")
    ps.add_argument("--n", type=int, nargs="+", required=True)
    ps.add_argument("--model", default="m31")
    ps.add_argument("--seed", type=int, default=1)
    ps.add_argument("--steps", type=int, default=4)
    ps.add_argument("--eps", type=float, default=0.03125)
    ps.add_argument("--dacc-one", default="2^-9")
    ps.add_argument("--out", default="scaling.csv")
    a = ap.parse_args()
    accuracy(a) if a.cmd == "accuracy" else scaling(a)


if __name__ == "__main__":
    main()
