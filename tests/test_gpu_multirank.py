"""GPU: the sharded multi-rank step on one device.

Ranks shard the sink groups and exchange accelerations either through the
window/unpack path the NCCL mesh uses (LocalExchange transport) or through the
fused peer exchange (the walk kernel stores finished groups into the peers'
accumulators; in-process pointers, or CUDA IPC between two processes).  The
sharded run must equal the single-rank run: identical trees (redundant,
deterministic builds), summed events identical, and accelerations, positions
and velocities BIT-IDENTICAL: a group's task tree and its ordered combination do
not depend on which rank (or warp) walks it."""
import os
import subprocess
import sys
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world,mesh", [(2, "copy"), (3, "copy"), (2, "p2p"), (3, "p2p")])
def test_sharded_steps_match_single_rank(world, mesh):
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
    (g2.Simulation.set_mesh_local if mesh == "copy" else g2.Simulation.set_mesh_local_p2p)(sims)
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
    # whole-system groups were cut into slices, dealt round-robin to the ranks: the same
    # slices for any rank count, summed in slice order -- hence still bit-identical
    heavy, slices = ref.walk_slices()
    assert heavy > 0 and slices >= 2 * heavy, (heavy, slices)
    assert all(s.walk_slices() == (heavy, slices) for s in sims)
    a = ref.system()
    for s in sims:
        b = s.system()
        for k in ("acc", "pos", "vel", "acc_old_mag"):
            assert np.array_equal(getattr(b, k), getattr(a, k)), k
    if mesh == "p2p":
        # shards balanced by the previous step's per-group costs, the sliced whole-system
        # groups dealt by expected cost: the ranks' shares of the last step's interactions are near equal
        # (at this small N the 60 sliced groups carry a large share of the work; 2^22, 8 ranks: 1.03)
        work = np.array([o.events.interactions for o in out], float)
        assert work.max() / work.mean() < 1.05, work


@pytest.mark.slow
@pytest.mark.parametrize("world", [4, 8])
def test_eight_rank_mesh_bit_identical(world):
    """SURVEY §8e's correctness check at 4 and 8 ranks (in-process fused peer exchange on one B200, M31
    N = 2^20, all-active, rebuild every step): accelerations and the evolved state bit-identical to the
    single-rank run, the whole-system groups sliced the same way, events summed exactly."""
    import paper_1811_02761_b200 as g2
    from paper_1811_02761_b200.gravitree import sample_model
    m, p, v = sample_model("m31", 1 << 20, 1)
    params = g2.GravParams(1.0, 2.0 ** -5, 2.0 ** -9)
    scheme = g2.StepScheme(dt_max=1.0 / 64, adaptive=False)

    def make():
        s = g2.Simulation(g2.ParticleSystem(m, p, v), params, scheme)
        s.set_rebuild_every_step(True)
        return s

    ref = make()
    ref.init()
    sims = [make() for _ in range(world)]
    g2.Simulation.set_mesh_local_p2p(sims)
    for s in sims:
        s.init()
    r0s = [ref.step() for _ in range(2)]
    outs = run_mesh(sims, 2)
    for r0, out in zip(r0s, outs):
        assert sum(o.events.interactions for o in out) == r0.events.interactions
        assert sum(o.events.mac_evals for o in out) == r0.events.mac_evals
    assert ref.walk_slices()[1] > 0 and all(s.walk_slices() == ref.walk_slices() for s in sims)
    a = ref.system()
    for s in sims:
        b = s.system()
        for k in ("acc", "pos", "vel", "acc_old_mag"):
            assert np.array_equal(getattr(b, k), getattr(a, k)), k


def run_mesh(sims, steps):
    out = []
    for _ in range(steps):
        res = [None] * len(sims)

        def run(k):
            res[k] = sims[k].step()

        th = [threading.Thread(target=run, args=(k,)) for k in range(len(sims))]
        for t in th:
            t.start()
        for t in th:
            t.join()
        assert all(o is not None for o in res)
        out.append(res)
    return out


@pytest.mark.parametrize("world,mesh", [(2, "copy"), (3, "p2p")])
def test_autotuned_mesh_matches_single_rank(world, mesh):
    """Block steps with the reference's rebuild auto-tuner on a mesh: every rank must take
    the same rebuild decisions.  With the deterministic tuner clock the ranks feed their tuners the
    SUM of their modelled walk times = the single-rank value, so the mesh reproduces the single-rank
    run bit for bit, rebuild schedule included."""
    import paper_1811_02761_b200 as g2
    from paper_1811_02761_b200.gravitree import sample_model
    m, p, v = sample_model("m31", 60000, 3)
    params = g2.GravParams(1.0, 2.0 ** -5, 2.0 ** -9)

    def make():
        s = g2.Simulation(g2.ParticleSystem(m, p, v), params, g2.StepScheme(dt_max=1.0))
        s.set_tuner_model(4e13, 3e-12)  # cheap builds: the tuner shortens the interval (several rebuilds)
        return s

    ref = make()
    ref.init()
    sims = [make() for _ in range(world)]
    (g2.Simulation.set_mesh_local if mesh == "copy" else g2.Simulation.set_mesh_local_p2p)(sims)
    for s in sims:
        s.init()
    single = [ref.step() for _ in range(24)]
    multi = run_mesh(sims, 24)
    assert sum(r.rebuilt for r in single) >= 2  # the first build and one auto-tuned rebuild at least
    for r0, rs in zip(single, multi):
        assert all(r.rebuilt == r0.rebuilt and r.rebuild_interval == r0.rebuild_interval for r in rs)
        assert all(r.active == r0.active for r in rs)
    a = ref.system()
    for s in sims:
        b = s.system()
        for k in ("acc", "pos", "vel", "level"):
            assert np.array_equal(getattr(b, k), getattr(a, k)), k


def test_autotuned_mesh_measured_times_consistent():
    """With the default (CUDA-event) tuner clock the ranks agree on the max of their measured times:
    rebuild decisions and the evolved state are identical on every rank."""
    import paper_1811_02761_b200 as g2
    from paper_1811_02761_b200.gravitree import sample_model
    m, p, v = sample_model("m31", 60000, 4)
    sims = [g2.Simulation(g2.ParticleSystem(m, p, v), g2.GravParams(1.0, 2.0 ** -5, 2.0 ** -9),
                          g2.StepScheme(dt_max=1.0)) for _ in range(2)]
    g2.Simulation.set_mesh_local_p2p(sims)
    for s in sims:
        s.init()
    for rs in run_mesh(sims, 14):
        assert rs[0].rebuilt == rs[1].rebuilt and rs[0].rebuild_interval == rs[1].rebuild_interval
    a, b = sims[0].system(), sims[1].system()
    for k in ("acc", "pos", "vel", "level"):
        assert np.array_equal(getattr(a, k), getattr(b, k)), k


def test_nccl_one_rank_mesh():
    """The NCCL exchange through product code (g2_sim_set_mesh): a one-rank communicator runs the
    sharded step path -- host-side shard, ncclAllGather of the accumulator window, unpack kernel, and
    the tuner agreement's ncclAllReduce -- and equals the plain single-rank run bit for bit.  (NCCL
    refuses two ranks on one device; the multi-rank window/unpack logic is the LocalExchange tests'.)"""
    import paper_1811_02761_b200 as g2
    from paper_1811_02761_b200.gravitree import sample_model
    m, p, v = sample_model("m31", 60000, 6)
    params = g2.GravParams(1.0, 2.0 ** -5, 2.0 ** -9)
    a = g2.Simulation(g2.ParticleSystem(m, p, v), params, g2.StepScheme(dt_max=1.0))
    b = g2.Simulation(g2.ParticleSystem(m, p, v), params, g2.StepScheme(dt_max=1.0))
    for s in (a, b):
        s.set_tuner_model(4e13, 3e-10)
    b.set_mesh(0, 1, g2.nccl_unique_id())
    for s in (a, b):
        s.init()
    ra = [a.step() for _ in range(10)]
    rb = [b.step() for _ in range(10)]
    assert [r.rebuilt for r in ra] == [r.rebuilt for r in rb]
    assert [r.events.interactions for r in ra] == [r.events.interactions for r in rb]
    sa, sb = a.system(), b.system()
    for k in ("acc", "pos", "vel", "level"):
        assert np.array_equal(getattr(sa, k), getattr(sb, k)), k


def test_deterministic_accelerations():
    """Two walks of the same M31 2^20 system (all active, many donated subtrees) and a block-step
    run repeated: bit-identical accelerations (the reference is thread-count independent,
    parallel.hpp:16-19, test_perflab.cpp:123-148)."""
    import paper_1811_02761_b200 as g2
    from paper_1811_02761_b200.gravitree import sample_model
    m, p, v = sample_model("m31", 1 << 20, 1)
    params = g2.GravParams(1.0, 2.0 ** -5, 2.0 ** -9)
    s0 = g2.ParticleSystem(m, p, v)
    eng = g2.GravityEngine(params)
    eng.build(s0)
    eng.bootstrap(s0)
    accs = []
    for _ in range(3):
        s = g2.ParticleSystem(m, p, v, acc_old_mag=s0.acc_old_mag.copy())
        ev = eng.evaluate(s)
        accs.append((s.acc.copy(), ev))
    for a, ev in accs[1:]:
        assert np.array_equal(a, accs[0][0]) and ev == accs[0][1]
    runs = []
    for _ in range(2):
        sim = g2.Simulation(g2.ParticleSystem(m, p, v), params, g2.StepScheme(dt_max=1.0))
        sim.init()
        sim.set_fixed_rebuild_interval(2)
        for _ in range(6):
            sim.step()
        runs.append(sim.system())
    for k in ("acc", "pos", "vel", "level"):
        assert np.array_equal(getattr(runs[0], k), getattr(runs[1], k)), k
    # the phase overlap (calcNode's internal levels beside the group set-up on a side stream) only
    # schedules: the same run with every phase alone on the step's stream is bit-identical
    sim = g2.Simulation(g2.ParticleSystem(m, p, v), params, g2.StepScheme(dt_max=1.0))
    sim.set_phase_overlap(False)
    sim.init()
    sim.set_fixed_rebuild_interval(2)
    for _ in range(6):
        sim.step()
    alone = sim.system()
    for k in ("acc", "pos", "vel", "level"):
        assert np.array_equal(getattr(runs[0], k), getattr(alone, k)), k


def test_p2p_ipc_two_processes(tmp_path):
    """Two processes (one rank each, both on cuda:0) map each other's exchange buffers
    through CUDA IPC, exactly as one process per GPU would; handles travel over gloo."""
    import paper_1811_02761_b200 as g2
    from paper_1811_02761_b200.gravitree import sample_model
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29613", os.path.join(root, "tests", "p2p_ranks.py"),
           str(tmp_path)]
    subprocess.run(cmd, check=True, cwd=root, timeout=600)
    m, p, v = sample_model("m31", 100000, 5)
    ref = g2.Simulation(g2.ParticleSystem(m, p, v), g2.GravParams(1.0, 2.0 ** -5, 2.0 ** -9),
                        g2.StepScheme(dt_max=1.0 / 64, adaptive=False))
    ref.set_rebuild_every_step(True)
    ref.init()
    inter = 0
    for _ in range(3):
        inter = ref.step().events.interactions
    a = ref.system()
    got = [np.load(tmp_path / f"rank{r}.npz") for r in range(2)]
    assert sum(int(g["inter"]) for g in got) == inter
    for g in got:
        assert np.array_equal(g["acc"], a.acc) and np.array_equal(g["pos"], a.pos)


def test_p2p_peer_timeout(tmp_path):
    """A peer that never reaches the device-side exchange barrier (crashed, hung, diverged) makes
    the waiting rank's step raise ResourceError after G2_PEER_TIMEOUT_S instead of hanging the GPU."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29617", os.path.join(root, "tests", "p2p_ranks.py"),
           str(tmp_path), "stall"]
    env = dict(os.environ, G2_PEER_TIMEOUT_S="2")
    subprocess.run(cmd, check=True, cwd=root, env=env, timeout=600)
    outcome = (tmp_path / "stall.txt").read_text()
    assert outcome.startswith("ResourceError") and "exchange barrier" in outcome, outcome


def test_bench_two_ranks_one_device(tmp_path):
    """bench.py's N > 1 path (torchrun, fused peer exchange, max over ranks) end to end, both ranks on
    cuda:0 through the bench's one-device test mode (gloo process group)."""
    import json
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, G2_BENCH_ONE_DEVICE="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29617", os.path.join(root, "bench.py"), "--gpus", "2",
           "--particles", "262144", "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--no-paper"]
    r = subprocess.run(cmd, cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    line = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(line) == 1, r.stdout
    d = json.loads(line[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["e2e"]["value"] > 0
    assert d["config"]["exchange"].startswith("fused")
