"""Python mirror of gravitree's operator API over the g2 C-ABI (include/g2/capi.h).

Same names, argument meaning and error behaviour as the reference C++ API
(/root/reference/proj/core/include/gravitree): ``GravityEngine``
(engine.hpp:29-66), ``Simulation`` (integrator.hpp:54-91), the free functions
``direct_sum`` (gravity.hpp:40-43), ``block_level`` / ``predict``
(integrator.hpp:28-41), ``count_walk_ops`` / ``flops_estimate``
(op_counters.hpp:54-88) and ``force_error`` (gravity.hpp:47-53), and the
exception hierarchy of errors.hpp:8-23.  Every numerical call runs in the
sm_100a library ``_build/libg2.so``; there is no CPU fallback — importing
this module without the built library raises ImportError.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# G2_LIB_PATH: development override (A/B experiments with alternative builds)
LIB_PATH = os.environ.get("G2_LIB_PATH") or os.path.join(_HERE, "_build", "libg2.so")


# ---- errors (errors.hpp:8-23) ---------------------------------------------------
class DataError(RuntimeError):
    """gravitree::data_error — malformed input or broken invariant (status 3)."""


class ResourceError(RuntimeError):
    """gravitree::resource_error — a configured capacity was exhausted (status 4)."""


class SingularityError(DataError):
    """gravitree::singularity_error — zero separation with zero softening (status 5)."""


class InternalError(RuntimeError):
    """CUDA / internal failure (status 1)."""


_ERRORS = {1: InternalError, 3: DataError, 4: ResourceError, 5: SingularityError}


# ---- C structs --------------------------------------------------------------------
class _GravParams(C.Structure):
    _fields_ = [("G", C.c_double), ("eps", C.c_double), ("dacc", C.c_double)]


class _EngineConfig(C.Structure):
    _fields_ = [("leaf_cap", C.c_size_t), ("group_size", C.c_size_t), ("list_capacity", C.c_size_t),
                ("frontier_cap", C.c_size_t), ("count_ops", C.c_int), ("bootstrap_theta", C.c_double),
                ("bootstrap_direct_limit", C.c_size_t), ("threads", C.c_uint)]


class _Events(C.Structure):
    _fields_ = [("interactions", C.c_uint64), ("mac_evals", C.c_uint64), ("list_pushes", C.c_uint64)]


class _StepScheme(C.Structure):
    _fields_ = [("eta", C.c_double), ("dt_max", C.c_double), ("adaptive", C.c_int), ("fixed_level", C.c_int)]


class _TunerConfig(C.Structure):
    _fields_ = [("min_interval", C.c_size_t), ("max_interval", C.c_size_t), ("initial_interval", C.c_size_t)]


class _StepResult(C.Structure):
    _fields_ = [("walk_tree", C.c_double), ("calc_node", C.c_double), ("make_tree", C.c_double),
                ("predict", C.c_double), ("correct", C.c_double), ("events", _Events), ("active", C.c_size_t),
                ("rebuild_interval", C.c_size_t), ("rebuilt", C.c_int), ("wall_seconds", C.c_double)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `make -C paper_1811_02761_b200` "
                          "(or __graft_entry__.build()); there is no CPU fallback")
    lib = C.CDLL(LIB_PATH)
    lib.g2_last_error.restype = C.c_char_p
    lib.g2_engine_has_tree.restype = C.c_int
    lib.g2_p2p_handle_bytes.restype = C.c_size_t
    return lib


_lib = _load()


def lib():
    return _lib


def _chk(code):
    if code != 0:
        msg = _lib.g2_last_error().decode(errors="replace")
        raise _ERRORS.get(code, InternalError)(msg)


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _f64(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    if shape is not None:
        a = a.reshape(shape)
    return a


# ---- parameter dataclasses (defaults identical to the reference) ------------------
@dataclass
class GravParams:
    """GravParams (particle_system.hpp:53-57)."""
    G: float = 1.0
    eps: float = 0.0
    dacc: float = 2.0 ** -9

    def _c(self):
        return _GravParams(self.G, self.eps, self.dacc)


@dataclass
class EngineConfig:
    """EngineConfig (engine.hpp:14-23)."""
    leaf_cap: int = 8
    group_size: int = 32
    list_capacity: int = 1024
    frontier_cap: int = 0
    count_ops: bool = True
    bootstrap_theta: float = 0.5
    bootstrap_direct_limit: int = 65536
    threads: int = 0

    def _c(self):
        return _EngineConfig(self.leaf_cap, self.group_size, self.list_capacity, self.frontier_cap,
                             int(self.count_ops), self.bootstrap_theta, self.bootstrap_direct_limit, self.threads)


@dataclass
class StepScheme:
    """StepScheme (integrator.hpp:18-23)."""
    eta: float = 0.5
    dt_max: float = 0.0625
    adaptive: bool = True
    fixed_level: int = 0

    def _c(self):
        return _StepScheme(self.eta, self.dt_max, int(self.adaptive), self.fixed_level)


@dataclass
class TunerConfig:
    """TunerConfig (rebuild_tuner.hpp:9-13)."""
    min_interval: int = 1
    max_interval: int = 128
    initial_interval: int = 8

    def _c(self):
        return _TunerConfig(self.min_interval, self.max_interval, self.initial_interval)


@dataclass
class TraversalEvents:
    """TraversalEvents (op_counters.hpp:33-46)."""
    interactions: int = 0
    mac_evals: int = 0
    list_pushes: int = 0

    @classmethod
    def _from(cls, e: _Events):
        return cls(int(e.interactions), int(e.mac_evals), int(e.list_pushes))

    def __add__(self, o):
        return TraversalEvents(self.interactions + o.interactions, self.mac_evals + o.mac_evals,
                               self.list_pushes + o.list_pushes)


@dataclass
class PhaseTimings:
    walk_tree: float = 0.0
    calc_node: float = 0.0
    make_tree: float = 0.0
    predict: float = 0.0
    correct: float = 0.0

    def total(self):
        return self.walk_tree + self.calc_node + self.make_tree + self.predict + self.correct


@dataclass
class StepResult:
    """StepResult (integrator.hpp:43-50); phase times are CUDA-event seconds."""
    timings: PhaseTimings = field(default_factory=PhaseTimings)
    events: TraversalEvents = field(default_factory=TraversalEvents)
    active: int = 0
    rebuild_interval: int = 0
    rebuilt: bool = False
    wall_seconds: float = 0.0


@dataclass
class ParticleSystem:
    """ParticleSystem (particle_system.hpp:14-49) as numpy arrays (n,), (n,3)."""
    mass: np.ndarray
    pos: np.ndarray
    vel: np.ndarray = None
    acc: np.ndarray = None
    acc_old_mag: np.ndarray = None
    level: np.ndarray = None
    time: float = 0.0

    def __post_init__(self):
        n = len(self.mass)
        self.mass = _f64(self.mass)
        self.pos = _f64(self.pos, (n, 3))
        self.vel = np.zeros((n, 3)) if self.vel is None else _f64(self.vel, (n, 3))
        self.acc = np.zeros((n, 3)) if self.acc is None else _f64(self.acc, (n, 3))
        self.acc_old_mag = np.zeros(n) if self.acc_old_mag is None else _f64(self.acc_old_mag)
        self.level = np.zeros(n, np.uint8) if self.level is None else np.ascontiguousarray(self.level, np.uint8)

    def n(self):
        return len(self.mass)

    def copy(self):
        return ParticleSystem(self.mass.copy(), self.pos.copy(), self.vel.copy(), self.acc.copy(),
                              self.acc_old_mag.copy(), self.level.copy(), self.time)


@dataclass
class Tree:
    """Host copy of Octree (octree.hpp:32-42)."""
    bbox: np.ndarray
    keys: np.ndarray
    perm: np.ndarray
    rank: np.ndarray
    cells: np.ndarray  # (ncells, 4): first_child, child_count, first, count
    depth: np.ndarray
    nodes: np.ndarray  # (ncells, 5): mass, com xyz, extent


# ---- GravityEngine ------------------------------------------------------------------
class GravityEngine:
    """Tree-gravity driver on the B200 (engine.hpp:29-66).

    Mirrors the reference: build / build_structure / refresh / evaluate /
    bootstrap / tree / has_tree, with the system passed on every call.  The
    octree and all particle data live on the device between calls.
    """

    def __init__(self, params: GravParams = None, config: EngineConfig = None, device: int = 0):
        self._params = params or GravParams()
        self._config = config or EngineConfig()
        self._h = C.c_void_p()
        _chk(_lib.g2_engine_create(C.byref(self._params._c()), C.byref(self._config._c()), C.c_int(device),
                                   C.byref(self._h)))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            _lib.g2_engine_destroy(h)
            self._h = None

    @property
    def params(self):
        return self._params

    def set_params(self, p: GravParams):
        _chk(_lib.g2_engine_set_params(self._h, C.byref(p._c())))
        self._params = p

    @property
    def config(self):
        return self._config

    def build(self, system: ParticleSystem):
        _chk(_lib.g2_engine_build(self._h, C.c_size_t(system.n()), _ptr(system.mass), _ptr(system.pos)))

    def build_structure(self, system: ParticleSystem):
        _chk(_lib.g2_engine_build_structure(self._h, C.c_size_t(system.n()), _ptr(system.mass), _ptr(system.pos)))

    def refresh(self, system: ParticleSystem):
        _chk(_lib.g2_engine_refresh(self._h, C.c_size_t(system.n()), _ptr(system.mass), _ptr(system.pos)))

    def has_tree(self) -> bool:
        return bool(_lib.g2_engine_has_tree(self._h))

    def evaluate(self, system: ParticleSystem, targets=None, pot_out=None) -> TraversalEvents:
        """evaluate(system, targets, pot_out) — writes system.acc[targets] (engine.cpp:31-81)."""
        n = system.n()
        if pot_out is not None and len(pot_out) != n:
            raise DataError("GravityEngine::evaluate: potential span must cover the system")
        ev = _Events()
        tg = None
        nt = 0
        if targets is not None:
            tg = np.ascontiguousarray(targets, dtype=np.uint32)
            nt = len(tg)
            if nt == 0:  # engine.cpp:35: nothing to walk (a null pointer would mean "all" at the C ABI)
                if not self.has_tree():
                    raise DataError("GravityEngine::evaluate: no tree built")
                return TraversalEvents()
        pot = None
        if pot_out is not None:
            pot = np.ascontiguousarray(pot_out, dtype=np.float64)
        _chk(_lib.g2_engine_evaluate(self._h, C.c_size_t(n), _ptr(system.mass), _ptr(system.pos),
                                     _ptr(system.acc_old_mag), C.c_size_t(nt), _ptr(tg), _ptr(system.acc), _ptr(pot),
                                     C.byref(ev)))
        if pot_out is not None and pot is not pot_out:
            pot_out[:] = pot
        return TraversalEvents._from(ev)

    def bootstrap(self, system: ParticleSystem) -> TraversalEvents:
        """bootstrap(system) — direct sum for n <= bootstrap_direct_limit, else one geometric pass."""
        ev = _Events()
        _chk(_lib.g2_engine_bootstrap(self._h, C.c_size_t(system.n()), _ptr(system.mass), _ptr(system.pos),
                                      _ptr(system.acc), _ptr(system.acc_old_mag), C.byref(ev)))
        return TraversalEvents._from(ev)

    def tree(self) -> Tree:
        n, nc = C.c_size_t(), C.c_size_t()
        _chk(_lib.g2_engine_tree_size(self._h, C.byref(n), C.byref(nc)))
        n, nc = n.value, nc.value
        t = Tree(np.empty(4), np.empty(n, np.uint64), np.empty(n, np.uint32), np.empty(n, np.uint32),
                 np.empty((nc, 4), np.uint32), np.empty(nc, np.uint8), np.empty((nc, 5)))
        _chk(_lib.g2_engine_get_tree(self._h, _ptr(t.bbox), _ptr(t.keys), _ptr(t.perm), _ptr(t.rank), _ptr(t.cells),
                                     _ptr(t.depth), _ptr(t.nodes)))
        return t


# ---- Simulation -----------------------------------------------------------------------
class Simulation:
    """Block-time-step driver (integrator.hpp:54-91) with device-resident state."""

    def __init__(self, system: ParticleSystem, params: GravParams = None, scheme: StepScheme = None,
                 engine_config: EngineConfig = None, tuner_config: TunerConfig = None, device: int = 0):
        self._params = params or GravParams()
        self._scheme = scheme or StepScheme()
        self._n = system.n()
        self._mass = system.mass.copy()
        self._h = C.c_void_p()
        _chk(_lib.g2_sim_create(C.c_size_t(self._n), _ptr(system.mass), _ptr(system.pos), _ptr(system.vel),
                                C.byref(self._params._c()), C.byref(self._scheme._c()),
                                C.byref((engine_config or EngineConfig())._c()),
                                C.byref((tuner_config or TunerConfig())._c()), C.c_int(device), C.byref(self._h)))
        self._initialized = False

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            _lib.g2_sim_destroy(h)
            self._h = None

    def init(self):
        _chk(_lib.g2_sim_init(self._h))
        self._initialized = True

    def initialized(self):
        return self._initialized

    def step(self) -> StepResult:
        r = _StepResult()
        _chk(_lib.g2_sim_step(self._h, C.byref(r)))
        return StepResult(PhaseTimings(r.walk_tree, r.calc_node, r.make_tree, r.predict, r.correct),
                          TraversalEvents._from(r.events), int(r.active), int(r.rebuild_interval), bool(r.rebuilt),
                          r.wall_seconds)

    def set_fixed_rebuild_interval(self, interval: int):
        _chk(_lib.g2_sim_set_fixed_rebuild_interval(self._h, C.c_size_t(interval)))

    @classmethod
    def from_snapshot(cls, path, dacc: float = 2.0 ** -9, scheme: StepScheme = None,
                      engine_config: EngineConfig = None, tuner_config: TunerConfig = None, device: int = 0):
        """Simulation over a snapshot (read into pinned memory and uploaded in the library), with
        GravParams(snapshot G, snapshot eps, dacc) as the reference CLI builds them."""
        self = cls.__new__(cls)
        info = [C.c_size_t(), C.c_double(), C.c_double(), C.c_double()]
        _chk(_lib.g2_snapshot_info(str(path).encode(), *[C.byref(x) for x in info]))
        self._params = GravParams(info[2].value, info[3].value, dacc)
        self._scheme = scheme or StepScheme()
        self._n = info[0].value
        self._h = C.c_void_p()
        _chk(_lib.g2_sim_create_from_snapshot(str(path).encode(), C.c_double(dacc), C.byref(self._scheme._c()),
                                              C.byref((engine_config or EngineConfig())._c()),
                                              C.byref((tuner_config or TunerConfig())._c()), C.c_int(device),
                                              C.byref(self._h)))
        snap = read_snapshot(path)  # masses for system() (the device holds them in Morton order)
        self._mass = snap.system.mass
        self._initialized = False
        return self

    def write_snapshot(self, path):
        """The device-resident state as an OCTF snapshot (time, G, eps of this simulation)."""
        _chk(_lib.g2_sim_write_snapshot(self._h, str(path).encode()))

    def tree(self) -> Tree:
        """engine().tree() (integrator.hpp:62): the octree of the last rebuild."""
        n, nc = C.c_size_t(), C.c_size_t()
        _chk(_lib.g2_sim_tree_size(self._h, C.byref(n), C.byref(nc)))
        n, nc = n.value, nc.value
        t = Tree(np.empty(4), np.empty(n, np.uint64), np.empty(n, np.uint32), np.empty(n, np.uint32),
                 np.empty((nc, 4), np.uint32), np.empty(nc, np.uint8), np.empty((nc, 5)))
        _chk(_lib.g2_sim_get_tree(self._h, _ptr(t.bbox), _ptr(t.keys), _ptr(t.perm), _ptr(t.rank), _ptr(t.cells),
                                  _ptr(t.depth), _ptr(t.nodes)))
        return t

    def set_rebuild_every_step(self, on: bool = True):
        _chk(_lib.g2_sim_set_rebuild_every_step(self._h, C.c_int(int(on))))

    def set_phase_overlap(self, on: bool = True):
        """Overlap independent step phases on side streams (default on; off: every phase alone)."""
        _chk(_lib.g2_sim_set_phase_overlap(self._h, C.c_int(int(on))))

    def set_tuner_model(self, flop_rate: float, build_seconds_per_particle: float = 0.0):
        """The rebuild tuner's clock: CUDA-event times (flop_rate <= 0) or the deterministic model
        walk = (27 I + 5 M) / flop_rate, build = build_seconds_per_particle x n (reproducible schedule)."""
        _chk(_lib.g2_sim_set_tuner_model(self._h, C.c_double(flop_rate), C.c_double(build_seconds_per_particle)))

    def tuner_interval(self) -> int:
        v = C.c_size_t()
        _chk(_lib.g2_sim_tuner_interval(self._h, C.byref(v)))
        return v.value

    def sort_stats(self) -> tuple:
        """(bucket sorts, radix fallbacks) of the rebuilds so far (diagnostics)."""
        a, b = C.c_ulonglong(), C.c_ulonglong()
        _chk(_lib.g2_sim_sort_stats(self._h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def walk_kernel_seconds(self) -> float:
        """Device seconds of the last step's walk kernel alone (CUDA events around its launch)."""
        t = C.c_double()
        _chk(_lib.g2_sim_walk_kernel_seconds(self._h, C.byref(t)))
        return t.value

    def walk_slices(self) -> tuple:
        """(whole-system groups cut into slices, slices over all ranks) of the last step's walk."""
        a, b = C.c_uint(), C.c_uint()
        _chk(_lib.g2_sim_walk_slices(self._h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def system(self) -> ParticleSystem:
        n = self._n
        pos, vel, acc = np.empty((n, 3)), np.empty((n, 3)), np.empty((n, 3))
        am, lv, t = np.empty(n), np.empty(n, np.uint8), C.c_double()
        _chk(_lib.g2_sim_get_state(self._h, _ptr(pos), _ptr(vel), _ptr(acc), _ptr(am), _ptr(lv), C.byref(t)))
        return ParticleSystem(self._mass.copy(), pos, vel, acc, am, lv, t.value)

    def time(self) -> float:
        t = C.c_double()
        _chk(_lib.g2_sim_get_state(self._h, None, None, None, None, None, C.byref(t)))
        return t.value

    def set_state(self, pos=None, vel=None):
        p = None if pos is None else _f64(pos, (self._n, 3))
        v = None if vel is None else _f64(vel, (self._n, 3))
        _chk(_lib.g2_sim_set_state(self._h, _ptr(p), _ptr(v)))

    def set_mesh(self, rank: int, world: int, unique_id: bytes):
        """Join an NCCL mesh (one process per GPU): walk only this rank's shard of sink groups."""
        buf = (C.c_ubyte * 128).from_buffer_copy(unique_id)
        _chk(_lib.g2_sim_set_mesh(self._h, C.c_int(rank), C.c_int(world), buf))

    @staticmethod
    def set_mesh_local(sims):
        """In-process mesh: sims[r] walks shard r and the accelerations are exchanged by
        device copies; step the sims concurrently (one Python thread each)."""
        arr = (C.c_void_p * len(sims))(*[s._h.value for s in sims])
        _chk(_lib.g2_sim_set_mesh_local(arr, C.c_int(len(sims))))

    def p2p_export(self, rank: int, world: int) -> bytes:
        """Fused peer exchange, step 1: allocate this rank's exchange buffers and return their
        CUDA IPC handles; gather every rank's handles (rank order) out of band."""
        buf = (C.c_ubyte * _lib.g2_p2p_handle_bytes())()
        _chk(_lib.g2_sim_p2p_export(self._h, C.c_int(rank), C.c_int(world), buf))
        return bytes(buf)

    def set_mesh_p2p(self, rank: int, world: int, handles):
        """Fused peer exchange, step 2: map the peers' buffers.  The walk then stores each
        finished group's accelerations straight into every peer (no collective)."""
        blob = b"".join(handles)
        buf = (C.c_ubyte * len(blob)).from_buffer_copy(blob)
        _chk(_lib.g2_sim_set_mesh_p2p(self._h, C.c_int(rank), C.c_int(world), buf))

    @staticmethod
    def set_mesh_local_p2p(sims):
        """In-process mesh with the fused peer exchange (the walk pushes into the other sims'
        accumulators); step the sims concurrently (one Python thread each)."""
        arr = (C.c_void_p * len(sims))(*[s._h.value for s in sims])
        _chk(_lib.g2_sim_set_mesh_local_p2p(arr, C.c_int(len(sims))))


def nccl_unique_id() -> bytes:
    buf = (C.c_ubyte * 128)()
    _chk(_lib.g2_nccl_unique_id(buf))
    return bytes(buf)


# ---- free functions -----------------------------------------------------------------------
def direct_sum(system: ParticleSystem, params: GravParams = None, device: int = 0) -> np.ndarray:
    """direct_sum (gravity.cpp:18-43) on the device, FP64, reference summation order."""
    p = params or GravParams()
    acc = np.empty((system.n(), 3))
    _chk(_lib.g2_direct_sum(C.c_size_t(system.n()), _ptr(system.mass), _ptr(system.pos), C.c_double(p.G),
                            C.c_double(p.eps), C.c_int(device), _ptr(acc)))
    return acc


def direct_sum_targets(system: ParticleSystem, targets, params: GravParams = None, device: int = 0) -> np.ndarray:
    """Direct summation onto `targets` only (FP64 on the device; accuracy oracle at large N)."""
    p = params or GravParams()
    tg = np.ascontiguousarray(targets, dtype=np.uint32)
    acc = np.empty((len(tg), 3))
    _chk(_lib.g2_direct_sum_targets(C.c_size_t(system.n()), _ptr(system.mass), _ptr(system.pos), C.c_double(p.G),
                                    C.c_double(p.eps), C.c_size_t(len(tg)), _ptr(tg), C.c_int(device), _ptr(acc)))
    return acc


@dataclass
class Snapshot:
    """Snapshot (snapshot.hpp:16-20): the system (with its time) and the G, eps stored with it."""
    system: ParticleSystem
    G: float = 1.0
    eps: float = 0.0


def read_snapshot(path) -> Snapshot:
    """read_snapshot (snapshot.cpp:97-121): DataError with the reference's byte-offset messages."""
    n, t, G, eps = C.c_size_t(), C.c_double(), C.c_double(), C.c_double()
    _chk(_lib.g2_snapshot_info(str(path).encode(), C.byref(n), C.byref(t), C.byref(G), C.byref(eps)))
    if 40 + 56 * n.value > os.path.getsize(path):  # untrusted count: fail before allocating n particles
        _chk(_lib.g2_read_snapshot(str(path).encode(), C.c_size_t(0), None, None, None, None, None, None, None))
    mass, pos, vel = np.empty(n.value), np.empty((n.value, 3)), np.empty((n.value, 3))
    _chk(_lib.g2_read_snapshot(str(path).encode(), C.c_size_t(n.value), _ptr(mass), _ptr(pos), _ptr(vel), None,
                               None, None, None))
    sysm = ParticleSystem(mass, pos, vel)
    sysm.time = t.value
    return Snapshot(sysm, G.value, eps.value)


def write_snapshot(path, system: ParticleSystem, params: GravParams = None):
    """write_snapshot (snapshot.cpp:65-95): atomic temp file + rename."""
    p = params or GravParams()
    _chk(_lib.g2_write_snapshot(str(path).encode(), C.c_size_t(system.n()), _ptr(system.mass), _ptr(system.pos),
                                _ptr(system.vel), C.c_double(system.time), C.byref(p._c())))


@dataclass
class Diagnostics:
    """Diagnostics (diagnostics.hpp:9-15)."""
    kinetic: float = 0.0
    potential: float = 0.0
    total: float = 0.0
    momentum: np.ndarray = field(default_factory=lambda: np.zeros(3))
    virial_ratio: float = 0.0


class _CDiag(C.Structure):
    _fields_ = [("kinetic", C.c_double), ("potential", C.c_double), ("total", C.c_double),
                ("momentum", C.c_double * 3), ("virial_ratio", C.c_double)]


def compute_diagnostics(system: ParticleSystem, params: GravParams = None, device: int = 0) -> Diagnostics:
    """compute_diagnostics (diagnostics.cpp:10-38) on the device: energies, momentum and virial ratio.
    The potential is an FP64 direct sum up to 2^17 particles, beyond that the reference's dacc = 2^-20
    tree walk (FP32 forces/potentials) with the system's acc_old_mag."""
    p = params or GravParams()
    d = _CDiag()
    _chk(_lib.g2_compute_diagnostics(C.c_size_t(system.n()), _ptr(system.mass), _ptr(system.pos), _ptr(system.vel),
                                     _ptr(system.acc_old_mag), C.byref(p._c()), C.c_int(device), C.byref(d)))
    return Diagnostics(d.kinetic, d.potential, d.total, np.array(list(d.momentum)), d.virial_ratio)


def block_level(acc_mag, scheme: StepScheme = None, eps: float = 0.0, device: int = 0):
    """block_level (integrator.cpp:21-33), vectorised over acc_mag, on the device."""
    a = np.atleast_1d(np.ascontiguousarray(acc_mag, dtype=np.float64))
    out = np.empty(len(a), np.int32)
    _chk(_lib.g2_block_level(C.c_size_t(len(a)), _ptr(a), C.byref((scheme or StepScheme())._c()), C.c_double(eps),
                             C.c_int(device), _ptr(out)))
    return int(out[0]) if np.ndim(acc_mag) == 0 else out


def predict(system: ParticleSystem, dt: float, device: int = 0):
    """predict (integrator.cpp:40-45) on the device; updates system.pos / system.vel in place."""
    _chk(_lib.g2_predict(C.c_size_t(system.n()), _ptr(system.pos), _ptr(system.vel), _ptr(system.acc),
                         C.c_double(dt), C.c_int(device)))


# ---- measurement convention (op_counters.hpp:50-63, op_counters.cpp:14-19) ---------------
INTERACTION_COST = dict(integer=0, fp_fma=9, fp_add=3, fp_mul=2, fp_rsqrt=1)
MAC_EVAL_COST = dict(integer=12, fp_fma=0, fp_add=2, fp_mul=3, fp_rsqrt=0)
LIST_PUSH_COST = dict(integer=4, fp_fma=0, fp_add=0, fp_mul=0, fp_rsqrt=0)


def count_walk_ops(ev: TraversalEvents) -> dict:
    out = {}
    for k in INTERACTION_COST:
        out[k] = (INTERACTION_COST[k] * ev.interactions + MAC_EVAL_COST[k] * ev.mac_evals
                  + LIST_PUSH_COST[k] * ev.list_pushes)
    return out


def walk_flops(ev: TraversalEvents) -> float:
    """Flop by the paper's convention: FMA 2, add/mul 1, rsqrt 4 (27 per interaction, 5 per MAC)."""
    c = count_walk_ops(ev)
    return 2.0 * c["fp_fma"] + c["fp_add"] + c["fp_mul"] + 4.0 * c["fp_rsqrt"]


def flops_estimate(ev: TraversalEvents, elapsed_seconds: float) -> float:
    if not elapsed_seconds > 0.0:
        raise DataError("flops_estimate: elapsed time must be positive")
    return walk_flops(ev) / elapsed_seconds


def predict_speedup(ops: dict, peak_ratio: float = 1.5) -> float:
    """predict_speedup (op_counters.cpp:7-12): peak_ratio * (I + F) / max(I, F), F = fma + add + mul."""
    f = float(ops["fp_fma"] + ops["fp_add"] + ops["fp_mul"])
    i = float(ops["integer"])
    if f == 0.0 and i == 0.0:
        raise DataError("predict_speedup: no counted instructions")
    return peak_ratio * (i + f) / max(i, f)


def force_error(acc, ref) -> dict:
    """Nearest-rank relative-error statistics (gravity.cpp:67-90)."""
    acc, ref = np.asarray(acc, np.float64), np.asarray(ref, np.float64)
    if acc.shape != ref.shape:
        raise DataError("force_error: length mismatch")
    rn = np.sqrt((ref * ref).sum(1))
    keep = rn != 0.0
    d = acc[keep] - ref[keep]
    err = np.sort(np.sqrt((d * d).sum(1)) / rn[keep])
    if len(err) == 0:
        return {"median": 0.0, "p99": 0.0, "max": 0.0, "excluded": int((~keep).sum())}

    def nr(p):
        k = int(np.ceil(p / 100.0 * len(err)))
        return float(err[k - 1 if k else 0])

    return {"median": nr(50.0), "p99": nr(99.0), "max": float(err[-1]), "excluded": int((~keep).sum())}


# ---- inputs: bit-identical restatement of the reference samplers (csrc/ics.cpp) ------------
def sample_model(name: str, n: int, seed: int = 1, threads: int = 0):
    """sample_model (models.cpp:442-460) -> (mass[n], pos[n,3], vel[n,3]), bit-identical to the
    reference's output for the same (name, n, seed); multithreaded where the stream allows."""
    mass, pos, vel = np.empty(n), np.empty((n, 3)), np.empty((n, 3))
    _lib.g2_ics_last_error.restype = C.c_char_p
    code = _lib.g2_sample_model(name.encode(), C.c_size_t(n), C.c_uint64(seed), C.c_uint(threads), _ptr(mass),
                                _ptr(pos), _ptr(vel))
    if code != 0:
        raise DataError(_lib.g2_ics_last_error().decode())
    return mass, pos, vel
