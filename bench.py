#!/usr/bin/env python3
"""Benchmark: GOTHIC-style octree gravity step on B200 (BASELINE.json metric).

Workload (BASELINE.json configs[2], the paper's headline case): M31-like model
N = 2^23 (reference sample_model("m31", N, seed 1), reproduced bit-identically
by the library's sampler), dacc = 2^-9, eps = 2^-5, leaf 8, group 32.  One
"step" is one ALL-ACTIVE full block step through the library's Simulation:
predict -> makeTree (bbox, keys, radix sort, split) -> calcNode -> walkTree
(all N sinks) -> correct, with the tree rebuilt every step.

  value   seconds per step, state resident in HBM, device time (CUDA events on
          the library's stream), max over ranks.  Lower is better.
  e2e     the same step through the public C-ABI with host buffers: pinned
          positions/velocities uploaded, accelerations read back every step.
  roofline  walkTree (the dominant kernel) in TFLOP/s by the reference's own
          convention (27 Flop / interaction, 5 / MAC evaluation) against the
          FP32 CUDA-core peak (148 SM x 128 lanes x 2 x f_max).

`--impl reference` times the reference's CPU implementation (oracle/_ref) of
the same step on this host's cores: full, unsampled all-active steps of the
reference's own stepping loop (integrator.cpp:97-164 with a rebuild every
step), same metric string, unit and config as this arm.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

EPS = 2.0 ** -5
DACC = 2.0 ** -9
PAPER_V100_S_PER_STEP = 3.3e-2  # PAPER.md:18,191 (block-step average, not all-active)


def parse():
    return parse_args_list(None)


def parse_args_list(argv):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="g2", choices=["g2", "reference"])
    ap.add_argument("--n", "--particles", dest="n", type=int, default=1 << 23)
    ap.add_argument("--model", default="m31")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-paper", action="store_true", help="skip the paper-protocol block-step run")
    ap.add_argument("--paper-steps", type=int, default=32)
    ap.add_argument("--exchange", default="p2p", choices=["p2p", "nccl"],
                    help="multi-GPU acceleration exchange: fused walk-epilogue P2P stores, or ncclAllGather")
    return ap.parse_args(argv)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("G2_BENCH_ONE_DEVICE"):  # testing only: every rank on cuda:0, gloo process group
        local = 0
    return rank, world, local


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons polled through NVML every ~5 ms while the
    timed region runs (nvidia-smi's fastest loop is too coarse for a sub-second region); without
    NVML the summary reports zero samples."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))

    def __init__(self, device):
        self.device, self.sm, self.reasons, self.max_mhz = device, [], set(), None
        self._stop = threading.Event()

    def _poll(self, nv, h):
        while not self._stop.is_set():
            try:
                self.sm.append(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                for name, attr in self.REASONS:
                    if r & getattr(nv, attr, 0):
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.005)

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[self.device]) if vis else self.device
            h = nv.nvmlDeviceGetHandleByIndex(idx)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            self.t = threading.Thread(target=self._poll, args=(nv, h), daemon=True)
            self.t.start()
        except Exception:  # noqa: BLE001
            self.t = None
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.t:
            self.t.join(timeout=2)

    def summary(self):
        return {"sm_mhz": float(np.median(self.sm)) if self.sm else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.sm), "how": "NVML poll every ~5 ms"}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {}


def fp32_peak_measured():
    """The FP32 CUDA-core peak measured on this GPU by tools/fp32_peak.cu (built by build() into
    _build/fp32_peak): the larger of scalar FFMA and packed FFMA2 throughput, TFLOP/s; None if absent."""
    exe = os.path.join(ROOT, "paper_1811_02761_b200", "_build", "fp32_peak")
    try:
        out = subprocess.run([exe], capture_output=True, text=True, timeout=60, check=True).stdout
        d = json.loads(out.strip().splitlines()[-1])
        return max(d["ffma_tflops"], d["ffma2_tflops"]), d
    except (OSError, subprocess.SubprocessError, ValueError, KeyError, IndexError):
        return None, None


def walk_traffic_per_launch():
    """dram bytes per walk launch from the committed ncu capture, if any."""
    p = os.path.join(ROOT, "profiles", "walk_traffic.json")  # from the committed ncu --set full capture
    try:
        with open(p) as f:
            return json.load(f).get("dram_bytes_per_launch")
    except OSError:
        return None


# ------------------------------------------------------------------------- CPU reference
DT_STEP = 1.0 / 16  # level-0 step of the bench scheme (StepScheme dt_max = 1/16, fixed_level 0)


def metric_name(args):
    """One metric string for both arms (the driver divides the two only when they match)."""
    return f"sec/step ({args.model} N={args.n} all-active full step)"


def cpu_reference_loop(mass, pos, vel, acc=None, amag=None, threads=0):
    """The reference's stepping loop on this host (oracle/refpy.RefLoop): every step is one full,
    UNSAMPLED all-active step through the reference's public API -- predict, build_structure +
    refresh, evaluate on all N, corrector (integrator.cpp:97-164 with a rebuild every step)."""
    from oracle.refpy import Ref, RefLoop
    ref = Ref()
    return ref, RefLoop(ref, mass, pos, vel, G=1.0, eps=EPS, dacc=DACC, threads=threads, acc=acc, acc_old_mag=amag)


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle.refpy import Ref
    threads = int(Ref().lib.gtref_resolve_threads(0))
    t0 = time.perf_counter()
    mass, pos, vel = Ref().sample_model(args.model, args.n, 1)
    t_ic = time.perf_counter() - t0
    t0 = time.perf_counter()
    _, loop = cpu_reference_loop(mass, pos, vel, threads=0)  # the reference's bootstrap (Simulation::init)
    t_boot = time.perf_counter() - t0
    for _ in range(args.warmup):
        loop.step(DT_STEP)
    times, last = [], None
    t_wall = time.perf_counter()
    for _ in range(args.steps):
        t0 = time.perf_counter()
        last = loop.step(DT_STEP)
        times.append(time.perf_counter() - t0)
    t_wall = time.perf_counter() - t_wall
    v = float(np.mean(times))
    desc = (f"reference (oracle/_ref, unmodified gravitree) stepping loop on {args.model} N={args.n}: "
            f"{args.steps} full all-active steps (predict, build_structure, refresh, evaluate on all N, "
            f"correct), no sampling; {threads} threads")
    print(json.dumps({
        "impl": "reference", "metric": metric_name(args), "value": v, "unit": "s/step",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": v * 1e3,
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args),
        "cpu_baseline": {"value": v, "unit": "s/step", "cores": threads, "kind": "reference", "sample": desc},
        "e2e": {"value": v, "unit": "s/step", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "timed_wall_seconds": t_wall, "setup_seconds": {"ic": t_ic, "bootstrap": t_boot},
        "phases_last_step": {k: last[k] for k in ("predict", "make_tree", "calc_node", "walk_tree", "correct")},
        "events_last_step": last["events"]}))


def workload_config(args):
    return {"workload": f"{args.model} N={args.n} all-active full step (predict+makeTree+calcNode+walkTree+correct, "
                        f"rebuild every step)", "model": args.model, "n": args.n, "dacc": DACC, "eps": EPS,
            "leaf_cap": 8, "group_size": 32, "parallelism": f"groups sharded over {dist_env()[1]} GPU(s)",
            "exchange": ("none" if dist_env()[1] == 1 else
                         "fused: walk-epilogue P2P stores into peer accumulators (CUDA IPC)"
                         if getattr(args, "exchange", "p2p") == "p2p" else "ncclAllGather"),
            "l2": "no flush: the resident state (~1 GB at 2^23) exceeds the 126 MB L2"}


def hbm_phases(sim, r, n, alone=None):
    """HBM roofline of the non-walk phases of one all-active step: algorithmic
    bytes per particle x N over the phase's CUDA-event time, against the measured copy peak.
    makeTree = bbox+keys 60 B + radix sort 8 + 24 x 8 passes + split 8 B x mean particle depth
    + 40 B x cells/N; calcNode 94 B; predict 120 B; correct 150 B per active particle."""
    peak = measured_peaks().get("hbm_gbs")
    t = sim.tree()
    leaf = t.cells[:, 1] == 0
    depth_mean = float((t.cells[leaf, 3].astype(np.float64) * t.depth[leaf]).sum() / n)
    per = {"make_tree": 60 + 8 + 24 * 8 + 8 * depth_mean + 40 * len(t.depth) / n, "calc_node": 94.0,
           "predict": 120.0, "correct": 150.0 * r.active / n}
    out = {"peak_gbs": peak, "peak_note": "MEASURED_PEAKS.json hbm_gbs (copy, read+write)",
           "mean_particle_depth": depth_mean, "cells_per_particle": len(t.depth) / n}
    for k, b in per.items():
        sec = getattr(r.timings, k)
        if alone and k in alone:
            # in the timed steps part of the phase runs on a side stream beside later phases, so its
            # span is not the phase's own time: the phase alone, measured in extra steps
            sec = alone[k]
        gbs = b * n / sec / 1e9 if sec > 0 else None
        out[k] = {"bytes_per_particle": b, "seconds": sec, "achieved_gbs": gbs,
                  "frac": gbs / peak if gbs and peak else None}
        if alone and k in alone:
            out[k]["how"] = ("3 extra all-active steps after the timed region with the phase overlap off (CUDA "
                             f"events); the span on the step's stream in the timed steps: {getattr(r.timings, k):.6f} s")
    return out


# ------------------------------------------------------------------------- g2 arm
def join_mesh(args, g2, sim, rank, world):
    """Shard the sink groups over the ranks.  p2p (default): the fused exchange -- the walk
    kernel stores each finished group's accelerations into every peer's buffer over NVLink
    (CUDA IPC handles all-gathered once at setup); nccl: one ncclAllGather per step."""
    import torch.distributed as dist
    if args.exchange == "p2p":
        handles = [None] * world
        err = None
        try:
            h = sim.p2p_export(rank, world)
        except Exception as e:  # noqa: BLE001
            h, err = None, e
        dist.all_gather_object(handles, h)
        if all(x is not None for x in handles):
            try:
                sim.set_mesh_p2p(rank, world, handles)
            except Exception as e:  # noqa: BLE001
                err = e
        ok = [None] * world
        dist.all_gather_object(ok, err is None)
        if all(ok):
            return
        # every rank falls back together (a mixed mesh would deadlock)
        print(f"[bench] rank {rank}: fused P2P exchange unavailable ({err}); using ncclAllGather", file=sys.stderr)
        args.exchange = "nccl"
    uid = [g2.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    sim.set_mesh(rank, world, uid[0])


def paper_protocol(args, g2, mass, pos, vel, params, local, rank, world, tuner_clock=None):
    """The paper-comparable block-step protocol: reference defaults
    (eta 0.5, adaptive levels) with dt_max = 1, timed over `paper_steps` steps after init and
    4 warm-up steps, once with the reference's own rebuild auto-tuner (fed CUDA-event times)
    and once with a fixed rebuild interval of 2 (the shortest the reference's tuner allows:
    GPU rebuilds are cheap); plus the reference's default scheme (dt_max = 1/16, auto-tuner), the
    other block-step scheme SURVEY §8d config 3 names.  Reports mean device s/step next to the paper's
    V100 3.3e-2 s/step, the mean active fraction and s per 1e11 walk Flop."""
    import ctypes
    import torch
    from paper_1811_02761_b200.gravitree import lib
    out = {"what": "block steps, reference driver defaults with dt_max=1 (eta 0.5, adaptive levels)",
           "paper_v100_s_per_step": PAPER_V100_S_PER_STEP,
           "tuner_clock": ("deterministic model calibrated on this run's all-active steps: walk %.2f TFLOP/s, "
                           "build %.3g s/particle (CUDA-event times make the reference's tuner schedule "
                           "timing-dependent: 6.8-32 ms/step across runs)" % (tuner_clock[0] / 1e12, tuner_clock[1])
                           if tuner_clock else "CUDA-event times")}
    for label, fixed, dt_max in (("auto_tuned_rebuild", 0, 1.0), ("rebuild_every_2", 2, 1.0),
                                 ("default_scheme_dt_max_1_16_auto_tuned", 0, 1.0 / 16)):
        sim = g2.Simulation(g2.ParticleSystem(mass, pos, vel), params, g2.StepScheme(eta=0.5, dt_max=dt_max),
                            g2.EngineConfig(), device=local)
        if world > 1:
            join_mesh(args, g2, sim, rank, world)
        sim.init()
        if fixed:
            sim.set_fixed_rebuild_interval(fixed)
        elif tuner_clock:
            sim.set_tuner_model(*tuner_clock)
        hs = ctypes.c_void_p()
        lib().g2_sim_stream(sim._h, ctypes.byref(hs))
        stream = torch.cuda.ExternalStream(hs.value, device=torch.device("cuda", local))
        for _ in range(4):
            sim.step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        rs = []
        with ClockSampler(local) as clk:  # the block steps run long after the headline region: clocks too
            e0.record(stream)
            for _ in range(args.paper_steps):
                rs.append(sim.step())
            e1.record(stream)
            e1.synchronize()
        s_per_step = e0.elapsed_time(e1) / 1e3 / args.paper_steps
        # the phases' own CUDA-event spans; the rest of the step span is device idle between the
        # phases and between steps (host round trips, launch latency)
        phase_s = float(np.mean([r.timings.total() for r in rs]))
        phase_split = {k: float(np.mean([getattr(r.timings, k) for r in rs]))
                       for k in ("predict", "make_tree", "calc_node", "walk_tree", "correct")}
        flops = float(np.mean([g2.walk_flops(r.events) for r in rs]))
        if world > 1:
            import torch.distributed as dist
            t = torch.tensor([s_per_step], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            s_per_step = float(t[0])
            t = torch.tensor([flops], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.SUM)
            flops = float(t[0])
        out[label] = {"steps": args.paper_steps, "dt_max": dt_max, "s_per_step": s_per_step,
                      "mean_active_fraction": float(np.mean([r.active for r in rs])) / args.n,
                      "rebuilds": int(sum(r.rebuilt for r in rs)), "walk_flop_per_step": flops,
                      "clocks": clk.summary(), "phases_s_per_step": phase_split,
                      "outside_phases_s_per_step": s_per_step - phase_s,
                      "speedup_vs_paper_v100": PAPER_V100_S_PER_STEP / s_per_step if s_per_step > 0 else None,
                      "s_per_1e11_walk_flop": s_per_step / (flops / 1e11) if flops > 0 else None}
        del sim
    return out


def run_g2(args):
    rank, world, local = dist_env()
    import torch
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        if os.environ.get("G2_BENCH_ONE_DEVICE"):
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_1811_02761_b200 as g2
    from paper_1811_02761_b200.gravitree import lib, sample_model

    # the walk's roofline denominator, measured on this GPU (rank 0, before anything is timed)
    fp32_meas, fp32_meas_d = fp32_peak_measured() if rank == 0 else (None, None)
    mass, pos, vel = sample_model(args.model, args.n, 1)
    params = g2.GravParams(1.0, EPS, DACC)
    scheme = g2.StepScheme(eta=0.5, dt_max=1.0 / 16, adaptive=False, fixed_level=0)  # every particle active
    sim = g2.Simulation(g2.ParticleSystem(mass, pos, vel), params, scheme, g2.EngineConfig(), device=local)
    sim.set_rebuild_every_step(True)
    if world > 1:
        join_mesh(args, g2, sim, rank, world)
    t0 = time.perf_counter()
    sim.init()
    t_init = time.perf_counter() - t0
    import ctypes
    hs = ctypes.c_void_p()
    lib().g2_sim_stream(sim._h, ctypes.byref(hs))
    stream = torch.cuda.ExternalStream(hs.value, device=torch.device("cuda", local))

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        sim.step()
    barrier()
    lib().g2_launch_count.restype = ctypes.c_ulonglong
    l0 = lib().g2_launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    results, walk_kernel = [], []
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            results.append(sim.step())
            walk_kernel.append(sim.walk_kernel_seconds())  # events around the walk kernel (step already synced)
        ev1.record(stream)
        ev1.synchronize()
    launches = (lib().g2_launch_count() - l0) / args.steps
    # makeTree's and calcNode's own kernels: the timed steps overlap the rebuild's reorder of the
    # corrector's state and calcNode's internal levels with later phases (side streams)
    sim.set_phase_overlap(False)
    alone_steps = [sim.step().timings for _ in range(3)]
    sim.set_phase_overlap(True)
    alone = {k: float(np.mean([getattr(t, k) for t in alone_steps])) for k in ("make_tree", "calc_node")}
    total_s = ev0.elapsed_time(ev1) / 1e3
    walk_s = float(np.mean([r.timings.walk_tree for r in results]))  # the phase: group set-up + kernel
    walk_kernel_s = float(np.mean(walk_kernel))
    per_step = total_s / args.steps
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([per_step, walk_s, walk_kernel_s], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        per_step, walk_s, walk_kernel_s = float(t[0]), float(t[1]), float(t[2])
    r0 = results[-1]
    flops = g2.walk_flops(r0.events)
    if world > 1:  # each rank counted its own shard of the groups
        import torch.distributed as dist
        t = torch.tensor([flops], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        flops = float(t[0])
    peaks = measured_peaks()
    f_max = float(peaks.get("sm_max_mhz", 1965.0))
    fp32_peak = 148 * 128 * 2 * f_max * 1e6 / 1e12  # TFLOP/s (nominal fallback)
    peak_note = (f"nominal: 148 SM x 128 FP32 lanes x 2 x {f_max:.0f} MHz (sm_max_mhz of MEASURED_PEAKS.json); "
                 "the FP32 micro-benchmark was not available")
    if fp32_meas:
        fp32_peak = fp32_meas
        peak_note = (f"measured on this GPU before the timed region by tools/fp32_peak.cu (max of scalar FFMA "
                     f"{fp32_meas_d['ffma_tflops']} and packed FFMA2 {fp32_meas_d['ffma2_tflops']} TFLOP/s; nominal "
                     f"{148 * 128 * 2 * f_max * 1e6 / 1e12:.2f})")
    achieved = flops / walk_kernel_s / 1e12 if walk_kernel_s > 0 else 0.0
    clocks = clk.summary()

    # e2e: through the public API with host buffers (pinned), copies in the timed region
    e2e = None
    if not args.no_e2e:
        hpos = torch.empty((args.n, 3), dtype=torch.float64, pin_memory=True).numpy()
        hvel = torch.empty((args.n, 3), dtype=torch.float64, pin_memory=True).numpy()
        hacc = torch.empty((args.n, 3), dtype=torch.float64, pin_memory=True).numpy()
        st = sim.system()
        hpos[:], hvel[:] = st.pos, st.vel
        hp = hacc.ctypes.data_as(ctypes.c_void_p)
        k = max(2, args.steps // 2)

        def e2e_step():
            sim.set_state(hpos, hvel)
            sim.step()
            lib().g2_sim_get_state(sim._h, None, None, hp, None, None, None)

        for _ in range(max(2, args.warmup)):  # untimed: first-touch of the staging buffers and pinned pages
            e2e_step()
        barrier()
        t0 = time.perf_counter()
        for _ in range(k):
            e2e_step()
        barrier()
        e2e_s = (time.perf_counter() - t0) / k
        if world > 1:
            import torch.distributed as dist
            t = torch.tensor([e2e_s], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t[0])
        e2e = {"value": e2e_s, "unit": "s/step", "h2d_bytes_per_step": int(hpos.nbytes + hvel.nbytes),
               "d2h_bytes_per_step": int(hacc.nbytes),
               "how": "host wall clock around set_state(pinned pos, vel) + step + get acc, per step"}

    paper = None
    if not args.no_paper:
        # the auto-tuned runs' tuner clock: the deterministic model calibrated on this run's all-active
        # steps (walk Flop rate, build seconds per particle), so the rebuild schedule is reproducible
        build_pp = float(np.mean([r.timings.make_tree + r.timings.calc_node for r in results])) / args.n
        if world > 1:  # every rank's tuner must see the same clock (collective rebuild decisions)
            import torch.distributed as dist
            t = torch.tensor([build_pp], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            build_pp = float(t[0])
        # rounded to two digits: run-to-run timing noise must not move a tuner decision
        paper = paper_protocol(args, g2, mass, pos, vel, params, local, rank, world,
                               tuner_clock=(float(f"{achieved * 1e12:.2g}"), float(f"{build_pp:.2g}")))

    hbm = hbm_phases(sim, r0, args.n, alone) if rank == 0 else None

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            # one full, unsampled all-active step of the reference on the same input (~20 s on the
            # box's 16 cores); the held accelerations come from the g2 state so no bootstrap runs
            st = sim.system()
            ref, loop = cpu_reference_loop(mass, pos, vel, acc=st.acc, amag=st.acc_old_mag)
            ph = loop.step(DT_STEP)
            cpu = {"value": ph["total"], "unit": "s/step", "cores": int(ref.lib.gtref_resolve_threads(0)),
                   "kind": "reference",
                   "sample": f"oracle/_ref (unmodified reference library): ONE full all-active step (predict, "
                             f"build_structure, refresh, evaluate on all N={args.n}, correct) on the same "
                             f"{args.model} input, no sampling",
                   "phases": {k: ph[k] for k in ("predict", "make_tree", "calc_node", "walk_tree", "correct")},
                   "events": ph["events"]}
            del loop
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "unit": "s/step", "cores": 0, "kind": "reference", "sample": f"unavailable: {e}"}

    if rank == 0:
        out = {
            "metric": metric_name(args), "value": per_step,
            "unit": "s/step", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": per_step * 1e3, "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32 walk / f64 tree+integrator", "data": "synthetic (reference sample_model m31, seed 1)",
            "config": workload_config(args),
            "roofline": {"bound": "fp32", "kernel": "walk_kernel", "achieved": achieved, "peak": fp32_peak,
                         "unit": "TFLOP/s", "frac": achieved / fp32_peak, "traffic": walk_traffic_per_launch() if (args.n == 1 << 23 and world == 1) else None,
                         "peak_note": peak_note,
                         "flop_per_launch": flops, "kernel_seconds": walk_kernel_s,
                         "kernel_seconds_how": "CUDA events around the walk kernel launch on its stream, mean of the timed steps",
                         "walk_phase_seconds": walk_s},
            "phases_last_step": vars(r0.timings), "events_last_step": vars(r0.events), "active": r0.active,
            "init_seconds": t_init, "e2e": e2e, "gpu_launches": launches * args.steps,
            "gpu_launches_per_step": launches, "clocks": clocks, "cpu_baseline": cpu,
            "paper_protocol": paper, "hbm_phases": hbm,
        }
        print(json.dumps(out))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_g2(args)


if __name__ == "__main__":
    main()
