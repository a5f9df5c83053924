"""ORACLE / TEST INFRASTRUCTURE ONLY — ctypes bindings for the two CPU checkers.

* ``Ref``    -> oracle/_ref/libgravitree_ref.so : the UNMODIFIED reference
               library (compiled in place from /root/reference by
               oracle/Makefile) behind the extern "C" shim oracle/ref_shim.cpp.
* ``Oracle`` -> oracle/_build/libg2oracle.so    : the plain-C restatement
               oracle/g2_oracle.c of the hot path.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs may import this module.  The product path
(paper_1811_02761_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libgravitree_ref.so")
ORACLE_SO = os.path.join(HERE, "_build", "libg2oracle.so")

_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_sz = C.c_size_t


class RefError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"status {code}: {msg}")
        self.code = code
        self.msg = msg


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _u32(a):
    return np.ascontiguousarray(a, dtype=np.uint32)


class Tree:
    """Host copy of an Octree (octree.hpp:32-42) in flat arrays."""

    def __init__(self, bbox, keys, perm, rank, cells, depth, nodes):
        self.bbox = bbox  # [cx, cy, cz, half]
        self.keys = keys  # u64[n]
        self.perm = perm  # u32[n]
        self.rank = rank  # u32[n]
        self.cells = cells  # u32[ncells, 4]: first_child, child_count, first, count
        self.depth = depth  # u8[ncells]
        self.nodes = nodes  # f64[ncells, 5]: mass, com xyz, extent


class Ref:
    """The reference library (oracle/_ref)."""

    _lib = None

    def __init__(self, path: str = REF_SO):
        if Ref._lib is None:
            if not os.path.exists(path):
                raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where /root/reference exists")
            lib = C.CDLL(path)
            lib.gtref_last_error.restype = C.c_char_p
            lib.gtref_tree_ncells.restype = _sz
            lib.gtref_engine_ncells.restype = _sz
            lib.gtref_autotune.restype = _sz
            lib.gtref_resolve_threads.restype = C.c_uint
            lib.gtref_block_level.restype = C.c_int
            lib.gtref_block_level.argtypes = [C.c_double, C.c_double, C.c_double, C.c_int, C.c_int, C.c_double]
            Ref._lib = lib
        self.lib = Ref._lib

    def _chk(self, code):
        if code != 0:
            raise RefError(code, self.lib.gtref_last_error().decode())

    # -- inputs ------------------------------------------------------------
    def sample_model(self, name: str, n: int, seed: int = 1):
        mass = np.empty(n)
        pos = np.empty((n, 3))
        vel = np.empty((n, 3))
        self._chk(self.lib.gtref_sample_model(name.encode(), _sz(n), C.c_uint64(seed),
                                              mass.ctypes.data_as(C.c_void_p), pos.ctypes.data_as(C.c_void_p),
                                              vel.ctypes.data_as(C.c_void_p)))
        return mass, pos, vel

    # -- trees ---------------------------------------------------------------
    def _get_tree(self, getter, h, n, ncells):
        bbox = np.empty(4)
        keys = np.empty(n, np.uint64)
        perm = np.empty(n, np.uint32)
        rank = np.empty(n, np.uint32)
        cells = np.empty((ncells, 4), np.uint32)
        depth = np.empty(ncells, np.uint8)
        nodes = np.zeros((ncells, 5))
        getter(h, *(a.ctypes.data_as(C.c_void_p) for a in (bbox, keys, perm, rank, cells, depth, nodes)))
        return Tree(bbox, keys, perm, rank, cells, depth, nodes)

    def build_tree(self, mass, pos, leaf_cap: int = 8, with_nodes: bool = True) -> Tree:
        mass, pos = _f64(mass), _f64(pos)
        h = C.c_void_p()
        self._chk(self.lib.gtref_tree_build(_sz(len(mass)), mass.ctypes.data_as(C.c_void_p),
                                            pos.ctypes.data_as(C.c_void_p), _sz(leaf_cap), C.c_int(int(with_nodes)),
                                            C.byref(h)))
        try:
            nc = self.lib.gtref_tree_ncells(h)
            return self._get_tree(self.lib.gtref_tree_get, h, len(mass), nc)
        finally:
            self.lib.gtref_tree_free(h)

    def calc_node_on(self, mass_build, pos_build, mass, pos, leaf_cap=8) -> Tree:
        """build_tree(pos_build) then calc_node(pos) — the stale-topology refresh."""
        mb, pb, m, p = _f64(mass_build), _f64(pos_build), _f64(mass), _f64(pos)
        h = C.c_void_p()
        self._chk(self.lib.gtref_tree_build(_sz(len(mb)), mb.ctypes.data_as(C.c_void_p), pb.ctypes.data_as(C.c_void_p),
                                            _sz(leaf_cap), C.c_int(0), C.byref(h)))
        try:
            self._chk(self.lib.gtref_tree_calc_node(h, _sz(len(m)), m.ctypes.data_as(C.c_void_p),
                                                    p.ctypes.data_as(C.c_void_p), C.c_uint(1)))
            nc = self.lib.gtref_tree_ncells(h)
            return self._get_tree(self.lib.gtref_tree_get, h, len(m), nc)
        finally:
            self.lib.gtref_tree_free(h)

    def bounding_cube(self, pos):
        pos = _f64(pos)
        out = np.empty(4)
        self._chk(self.lib.gtref_bounding_cube(_sz(len(pos)), pos.ctypes.data_as(C.c_void_p),
                                               out.ctypes.data_as(C.c_void_p)))
        return out

    # -- engine ----------------------------------------------------------------
    def engine(self, G=1.0, eps=0.0, dacc=2.0 ** -9, leaf_cap=8, group_size=32, list_capacity=1024,
               frontier_cap=0, count_ops=True, theta=0.5, direct_limit=65536, threads=0):
        return RefEngine(self, G, eps, dacc, leaf_cap, group_size, list_capacity, frontier_cap, count_ops, theta,
                         direct_limit, threads)

    def direct_sum(self, mass, pos, G=1.0, eps=0.0, threads=0):
        mass, pos = _f64(mass), _f64(pos)
        acc = np.empty_like(pos)
        self._chk(self.lib.gtref_direct_sum(_sz(len(mass)), mass.ctypes.data_as(C.c_void_p),
                                            pos.ctypes.data_as(C.c_void_p), C.c_double(G), C.c_double(eps),
                                            C.c_uint(threads), acc.ctypes.data_as(C.c_void_p)))
        return acc

    def write_snapshot(self, path, mass, pos, vel, time=0.0, G=1.0, eps=0.0):
        mass, pos, vel = _f64(mass), _f64(pos), _f64(vel)
        self._chk(self.lib.gtref_write_snapshot(str(path).encode(), _sz(len(mass)), mass.ctypes.data_as(C.c_void_p),
                                                pos.ctypes.data_as(C.c_void_p), vel.ctypes.data_as(C.c_void_p),
                                                C.c_double(time), C.c_double(G), C.c_double(eps)))

    def read_snapshot(self, path):
        """-> (mass, pos, vel, time, G, eps); raises DataError with the reference's message."""
        hdr = np.zeros(4)
        self._chk(self.lib.gtref_read_snapshot(str(path).encode(), _sz(0), None, None, None,
                                               hdr.ctypes.data_as(C.c_void_p)))
        n = int(hdr[0])
        mass, pos, vel = np.empty(n), np.empty((n, 3)), np.empty((n, 3))
        self._chk(self.lib.gtref_read_snapshot(str(path).encode(), _sz(n), mass.ctypes.data_as(C.c_void_p),
                                               pos.ctypes.data_as(C.c_void_p), vel.ctypes.data_as(C.c_void_p),
                                               hdr.ctypes.data_as(C.c_void_p)))
        return mass, pos, vel, hdr[1], hdr[2], hdr[3]

    def diagnostics(self, mass, pos, vel, acc_old_mag=None, G=1.0, eps=0.0, dacc=2.0 ** -9, threads=0):
        """compute_diagnostics (diagnostics.cpp:10-38) of the reference library."""
        mass, pos, vel = _f64(mass), _f64(pos), _f64(vel)
        am = None if acc_old_mag is None else _f64(acc_old_mag)
        out = np.empty(7)
        self._chk(self.lib.gtref_diagnostics(_sz(len(mass)), mass.ctypes.data_as(C.c_void_p),
                                             pos.ctypes.data_as(C.c_void_p), vel.ctypes.data_as(C.c_void_p),
                                             None if am is None else am.ctypes.data_as(C.c_void_p),
                                             C.c_double(G), C.c_double(eps), C.c_double(dacc), C.c_uint(threads),
                                             out.ctypes.data_as(C.c_void_p)))
        return {"kinetic": out[0], "potential": out[1], "total": out[2], "momentum": out[3:6].copy(),
                "virial_ratio": out[6]}

    def force_error(self, acc, ref):
        acc, ref = _f64(acc), _f64(ref)
        out = np.empty(4)
        self._chk(self.lib.gtref_force_error(_sz(len(acc)), acc.ctypes.data_as(C.c_void_p),
                                             ref.ctypes.data_as(C.c_void_p), out.ctypes.data_as(C.c_void_p)))
        return {"median": out[0], "p99": out[1], "max": out[2], "excluded": int(out[3])}

    def groups(self, pos, acc_old_mag, rank, targets, group_size=32):
        pos, am, rank, targets = _f64(pos), _f64(acc_old_mag), _u32(rank), _u32(targets)
        ng = (len(targets) + group_size - 1) // group_size
        out = np.empty((ng, 5))
        self._chk(self.lib.gtref_groups(_sz(len(pos)), pos.ctypes.data_as(C.c_void_p), am.ctypes.data_as(C.c_void_p),
                                        rank.ctypes.data_as(C.c_void_p), _sz(len(targets)),
                                        targets.ctypes.data_as(C.c_void_p), _sz(group_size),
                                        out.ctypes.data_as(C.c_void_p)))
        return out

    # -- integrator ---------------------------------------------------------------
    def block_level(self, acc_mag, eta=0.5, dt_max=1 / 16, adaptive=True, fixed_level=0, eps=0.0):
        return self.lib.gtref_block_level(acc_mag, eta, dt_max, int(adaptive), fixed_level, eps)

    def predict(self, pos, vel, acc, dt):
        pos, vel, acc = _f64(pos).copy(), _f64(vel).copy(), _f64(acc)
        self._chk(self.lib.gtref_predict(_sz(len(pos)), pos.ctypes.data_as(C.c_void_p),
                                         vel.ctypes.data_as(C.c_void_p), acc.ctypes.data_as(C.c_void_p),
                                         C.c_double(dt)))
        return pos, vel

    def correct(self, vel, acc, acc_old_mag, new_acc, dt):
        vel, acc, am, na = _f64(vel).copy(), _f64(acc).copy(), _f64(acc_old_mag).copy(), _f64(new_acc)
        self._chk(self.lib.gtref_correct(_sz(len(vel)), vel.ctypes.data_as(C.c_void_p),
                                         acc.ctypes.data_as(C.c_void_p), am.ctypes.data_as(C.c_void_p),
                                         na.ctypes.data_as(C.c_void_p), C.c_double(dt)))
        return vel, acc, am

    def autotune(self, build_time, hist, min_i=1, max_i=128, initial=8):
        h = _f64(hist)
        return int(self.lib.gtref_autotune(C.c_double(build_time), _sz(len(h)), h.ctypes.data_as(C.c_void_p),
                                           _sz(min_i), _sz(max_i), _sz(initial)))

    def simulation(self, mass, pos, vel, G=1.0, eps=0.0, dacc=2.0 ** -9, eta=0.5, dt_max=1 / 16, adaptive=True,
                   fixed_level=0, leaf_cap=8, group_size=32, threads=0):
        return RefSimulation(self, mass, pos, vel, G, eps, dacc, eta, dt_max, adaptive, fixed_level, leaf_cap,
                             group_size, threads)


class RefEngine:
    def __init__(self, ref: Ref, *args):
        self.ref, self.lib = ref, ref.lib
        G, eps, dacc, leaf_cap, group_size, list_cap, frontier_cap, count_ops, theta, direct_limit, threads = args
        self.h = C.c_void_p()
        ref._chk(self.lib.gtref_engine_create(C.c_double(G), C.c_double(eps), C.c_double(dacc), _sz(leaf_cap),
                                              _sz(group_size), _sz(list_cap), _sz(frontier_cap), C.c_int(int(count_ops)),
                                              C.c_double(theta), _sz(direct_limit), C.c_uint(threads), C.byref(self.h)))

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.gtref_engine_destroy(self.h)
            self.h = None

    def build(self, mass, pos, with_nodes=True):
        mass, pos = _f64(mass), _f64(pos)
        self.n = len(mass)
        self.ref._chk(self.lib.gtref_engine_build(self.h, _sz(len(mass)), mass.ctypes.data_as(C.c_void_p),
                                                  pos.ctypes.data_as(C.c_void_p), C.c_int(int(with_nodes))))

    def refresh(self, mass, pos):
        mass, pos = _f64(mass), _f64(pos)
        self.ref._chk(self.lib.gtref_engine_refresh(self.h, _sz(len(mass)), mass.ctypes.data_as(C.c_void_p),
                                                    pos.ctypes.data_as(C.c_void_p)))

    def tree(self) -> Tree:
        nc = self.lib.gtref_engine_ncells(self.h)
        return self.ref._get_tree(self.lib.gtref_engine_get_tree, self.h, self.n, nc)

    def evaluate(self, mass, pos, acc_old_mag, targets=None, with_potential=False, acc_init=None):
        mass, pos, am = _f64(mass), _f64(pos), _f64(acc_old_mag)
        n = len(mass)
        acc = np.zeros((n, 3)) if acc_init is None else _f64(acc_init).copy()
        pot = np.zeros(n) if with_potential else None
        ev = np.zeros(3, np.uint64)
        tp = None
        nt = 0
        if targets is not None:
            t = _u32(targets)
            tp, nt = t.ctypes.data_as(C.c_void_p), len(t)
        self.ref._chk(self.lib.gtref_engine_evaluate(self.h, _sz(n), mass.ctypes.data_as(C.c_void_p),
                                                     pos.ctypes.data_as(C.c_void_p), am.ctypes.data_as(C.c_void_p),
                                                     _sz(nt), tp, acc.ctypes.data_as(C.c_void_p),
                                                     pot.ctypes.data_as(C.c_void_p) if pot is not None else None,
                                                     ev.ctypes.data_as(C.c_void_p)))
        return acc, pot, {"interactions": int(ev[0]), "mac_evals": int(ev[1]), "list_pushes": int(ev[2])}

    def bootstrap(self, mass, pos):
        mass, pos = _f64(mass), _f64(pos)
        n = len(mass)
        self.n = n
        acc = np.empty((n, 3))
        am = np.empty(n)
        ev = np.zeros(3, np.uint64)
        self.ref._chk(self.lib.gtref_engine_bootstrap(self.h, _sz(n), mass.ctypes.data_as(C.c_void_p),
                                                      pos.ctypes.data_as(C.c_void_p), acc.ctypes.data_as(C.c_void_p),
                                                      am.ctypes.data_as(C.c_void_p), ev.ctypes.data_as(C.c_void_p)))
        return acc, am, {"interactions": int(ev[0]), "mac_evals": int(ev[1]), "list_pushes": int(ev[2])}


class RefSimulation:
    def __init__(self, ref: Ref, mass, pos, vel, G, eps, dacc, eta, dt_max, adaptive, fixed_level, leaf_cap,
                 group_size, threads):
        self.ref, self.lib = ref, ref.lib
        mass, pos, vel = _f64(mass), _f64(pos), _f64(vel)
        self.n = len(mass)
        self.h = C.c_void_p()
        ref._chk(self.lib.gtref_sim_create(_sz(self.n), mass.ctypes.data_as(C.c_void_p), pos.ctypes.data_as(C.c_void_p),
                                           vel.ctypes.data_as(C.c_void_p), C.c_double(G), C.c_double(eps),
                                           C.c_double(dacc), C.c_double(eta), C.c_double(dt_max), C.c_int(int(adaptive)),
                                           C.c_int(fixed_level), _sz(leaf_cap), _sz(group_size), C.c_uint(threads),
                                           C.byref(self.h)))

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.gtref_sim_destroy(self.h)
            self.h = None

    def init(self):
        self.ref._chk(self.lib.gtref_sim_init(self.h))

    def set_fixed_rebuild_interval(self, k):
        self.ref._chk(self.lib.gtref_sim_set_fixed_rebuild_interval(self.h, _sz(k)))

    def step(self):
        out = np.zeros(8)
        rebuilt = C.c_int()
        ev = np.zeros(3, np.uint64)
        self.ref._chk(self.lib.gtref_sim_step(self.h, out.ctypes.data_as(C.c_void_p), C.byref(rebuilt),
                                              ev.ctypes.data_as(C.c_void_p)))
        return {"walk_tree": out[0], "calc_node": out[1], "make_tree": out[2], "predict": out[3], "correct": out[4],
                "wall_seconds": out[5], "active": int(out[6]), "rebuild_interval": int(out[7]),
                "rebuilt": bool(rebuilt.value),
                "events": {"interactions": int(ev[0]), "mac_evals": int(ev[1]), "list_pushes": int(ev[2])}}

    def state(self):
        n = self.n
        pos, vel, acc = np.empty((n, 3)), np.empty((n, 3)), np.empty((n, 3))
        am = np.empty(n)
        lv = np.empty(n, np.uint8)
        t = C.c_double()
        self.lib.gtref_sim_get_state(self.h, pos.ctypes.data_as(C.c_void_p), vel.ctypes.data_as(C.c_void_p),
                                     acc.ctypes.data_as(C.c_void_p), am.ctypes.data_as(C.c_void_p),
                                     lv.ctypes.data_as(C.c_void_p), C.byref(t))
        return {"pos": pos, "vel": vel, "acc": acc, "acc_old_mag": am, "level": lv, "time": t.value}


class RefLoop:
    """All-active stepping loop over the reference's public API (ref_shim.cpp gtref_loop_*):
    Simulation::step (integrator.cpp:97-164) with every particle at level 0 and a rebuild every
    step.  acc/acc_old_mag None: the reference's bootstrap runs at construction (untimed)."""

    def __init__(self, ref: Ref, mass, pos, vel, G=1.0, eps=0.0, dacc=2.0 ** -9, threads=0, acc=None,
                 acc_old_mag=None):
        self.ref, self.lib = ref, ref.lib
        mass, pos, vel = _f64(mass), _f64(pos), _f64(vel)
        self.n = len(mass)
        self.h = C.c_void_p()
        acc_p = _f64(acc).ctypes.data_as(C.c_void_p) if acc is not None else None
        self._keep = (_f64(acc) if acc is not None else None, _f64(acc_old_mag) if acc_old_mag is not None else None)
        am_p = self._keep[1].ctypes.data_as(C.c_void_p) if acc_old_mag is not None else None
        if acc is not None:
            acc_p = self._keep[0].ctypes.data_as(C.c_void_p)
        ref._chk(self.lib.gtref_loop_create(_sz(self.n), mass.ctypes.data_as(C.c_void_p),
                                            pos.ctypes.data_as(C.c_void_p), vel.ctypes.data_as(C.c_void_p),
                                            acc_p, am_p, C.c_double(G), C.c_double(eps), C.c_double(dacc),
                                            C.c_uint(threads), C.byref(self.h)))
        self._keep = None

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.gtref_loop_destroy(self.h)
            self.h = None

    def step(self, dt):
        out = np.zeros(6)
        ev = np.zeros(3, np.uint64)
        self.ref._chk(self.lib.gtref_loop_step(self.h, C.c_double(dt), out.ctypes.data_as(C.c_void_p),
                                               ev.ctypes.data_as(C.c_void_p)))
        return {"predict": out[0], "make_tree": out[1], "calc_node": out[2], "walk_tree": out[3], "correct": out[4],
                "total": out[5],
                "events": {"interactions": int(ev[0]), "mac_evals": int(ev[1]), "list_pushes": int(ev[2])}}

    def state(self):
        n = self.n
        pos, vel, acc, am = np.empty((n, 3)), np.empty((n, 3)), np.empty((n, 3)), np.empty(n)
        self.lib.gtref_loop_get_state(self.h, pos.ctypes.data_as(C.c_void_p), vel.ctypes.data_as(C.c_void_p),
                                      acc.ctypes.data_as(C.c_void_p), am.ctypes.data_as(C.c_void_p))
        return {"pos": pos, "vel": vel, "acc": acc, "acc_old_mag": am}


class Oracle:
    """The plain-C restatement (oracle/g2_oracle.c), mirroring Ref's interface."""

    _lib = None

    def __init__(self, path: str = ORACLE_SO):
        if Oracle._lib is None:
            if not os.path.exists(path):
                raise FileNotFoundError(f"{path} missing: run `make -C oracle oracle`")
            lib = C.CDLL(path)
            lib.g2o_last_error.restype = C.c_char_p
            lib.g2o_tree_ncells.restype = _sz
            lib.g2o_autotune.restype = _sz
            lib.g2o_block_level.restype = C.c_int
            lib.g2o_block_level.argtypes = [C.c_double, C.c_double, C.c_double, C.c_int, C.c_int, C.c_double]
            Oracle._lib = lib
        self.lib = Oracle._lib

    def _chk(self, code):
        if code != 0:
            raise RefError(code, self.lib.g2o_last_error().decode())

    def bounding_cube(self, pos):
        pos = _f64(pos)
        out = np.empty(4)
        self._chk(self.lib.g2o_bounding_cube(_sz(len(pos)), pos.ctypes.data_as(C.c_void_p),
                                             out.ctypes.data_as(C.c_void_p)))
        return out

    def build_tree(self, mass, pos, leaf_cap=8, with_nodes=True, _keep=False):
        mass, pos = _f64(mass), _f64(pos)
        h = C.c_void_p()
        self._chk(self.lib.g2o_build_tree(_sz(len(mass)), mass.ctypes.data_as(C.c_void_p),
                                          pos.ctypes.data_as(C.c_void_p), _sz(leaf_cap), C.c_int(int(with_nodes)),
                                          C.byref(h)))
        n = len(mass)
        nc = self.lib.g2o_tree_ncells(h)
        bbox = np.empty(4)
        keys = np.empty(n, np.uint64)
        perm = np.empty(n, np.uint32)
        rank = np.empty(n, np.uint32)
        cells = np.empty((nc, 4), np.uint32)
        depth = np.empty(nc, np.uint8)
        nodes = np.zeros((nc, 5))
        self.lib.g2o_tree_get(h, *(a.ctypes.data_as(C.c_void_p) for a in (bbox, keys, perm, rank, cells, depth, nodes)))
        t = Tree(bbox, keys, perm, rank, cells, depth, nodes)
        if _keep:
            t._h = h
            t._mass, t._pos = mass, pos
        else:
            self.lib.g2o_tree_free(h)
        return t

    def calc_node_on(self, mass_build, pos_build, mass, pos, leaf_cap=8):
        """Topology from pos_build, node attributes from pos (stale-tree refresh)."""
        t = self.build_tree(mass_build, pos_build, leaf_cap, with_nodes=False, _keep=True)
        m, p = _f64(mass), _f64(pos)
        self.lib.g2o_calc_node(t._h, m.ctypes.data_as(C.c_void_p), p.ctypes.data_as(C.c_void_p))
        nodes = np.zeros((len(t.cells), 5))
        self.lib.g2o_tree_get(t._h, None, None, None, None, None, None, nodes.ctypes.data_as(C.c_void_p))
        self.lib.g2o_tree_free(t._h)
        t.nodes = nodes
        return t

    def evaluate(self, mass, pos, acc_old_mag, targets=None, G=1.0, eps=0.0, dacc=2.0 ** -9, leaf_cap=8,
                 group_size=32, list_capacity=1024, frontier_cap=0, theta=0.5, count_ops=True, threads=8,
                 with_potential=False, tree_pos=None, per_group=False):
        """Fresh build from tree_pos (default pos) then evaluate at pos; FP64."""
        mass, pos, am = _f64(mass), _f64(pos), _f64(acc_old_mag)
        n = len(mass)
        tp = pos if tree_pos is None else _f64(tree_pos)
        t = self.build_tree(mass, tp, leaf_cap, with_nodes=False, _keep=True)
        try:
            self.lib.g2o_calc_node(t._h, mass.ctypes.data_as(C.c_void_p), pos.ctypes.data_as(C.c_void_p))
            acc = np.zeros((n, 3))
            pot = np.zeros(n) if with_potential else None
            ev = np.zeros(3, np.uint64)
            tptr, nt = None, 0
            if targets is not None:
                tg = _u32(targets)
                tptr, nt = tg.ctypes.data_as(C.c_void_p), len(tg)
            ng = ((nt if targets is not None else n) + group_size - 1) // group_size
            gi = np.zeros(max(ng, 1), np.uint64) if per_group else None
            self._chk(self.lib.g2o_evaluate(t._h, _sz(n), mass.ctypes.data_as(C.c_void_p),
                                            pos.ctypes.data_as(C.c_void_p), am.ctypes.data_as(C.c_void_p), _sz(nt),
                                            tptr, C.c_double(G), C.c_double(eps), C.c_double(dacc), _sz(group_size),
                                            _sz(list_capacity), _sz(frontier_cap), C.c_double(theta),
                                            C.c_int(int(count_ops)), C.c_uint(threads), acc.ctypes.data_as(C.c_void_p),
                                            pot.ctypes.data_as(C.c_void_p) if pot is not None else None,
                                            ev.ctypes.data_as(C.c_void_p),
                                            gi.ctypes.data_as(C.c_void_p) if gi is not None else None))
        finally:
            self.lib.g2o_tree_free(t._h)
        events = {"interactions": int(ev[0]), "mac_evals": int(ev[1]), "list_pushes": int(ev[2])}
        if per_group:
            return acc, pot, events, gi[:ng]
        return acc, pot, events

    def groups(self, pos, acc_old_mag, rank, targets=None, group_size=32):
        pos, am, rank = _f64(pos), _f64(acc_old_mag), _u32(rank)
        nt = len(pos) if targets is None else len(targets)
        tg = None if targets is None else _u32(targets)
        out = np.empty(((nt + group_size - 1) // group_size, 5))
        self._chk(self.lib.g2o_groups(_sz(len(pos)), pos.ctypes.data_as(C.c_void_p), am.ctypes.data_as(C.c_void_p),
                                      rank.ctypes.data_as(C.c_void_p), _sz(nt),
                                      tg.ctypes.data_as(C.c_void_p) if tg is not None else None, _sz(group_size),
                                      out.ctypes.data_as(C.c_void_p)))
        return out

    def direct_sum(self, mass, pos, G=1.0, eps=0.0, threads=8):
        mass, pos = _f64(mass), _f64(pos)
        acc = np.empty_like(pos)
        self._chk(self.lib.g2o_direct_sum(_sz(len(mass)), mass.ctypes.data_as(C.c_void_p),
                                          pos.ctypes.data_as(C.c_void_p), C.c_double(G), C.c_double(eps),
                                          C.c_uint(threads), acc.ctypes.data_as(C.c_void_p)))
        return acc

    def block_level(self, acc_mag, eta=0.5, dt_max=1 / 16, adaptive=True, fixed_level=0, eps=0.0):
        return self.lib.g2o_block_level(acc_mag, eta, dt_max, int(adaptive), fixed_level, eps)

    def predict(self, pos, vel, acc, dt):
        pos, vel, acc = _f64(pos).copy(), _f64(vel).copy(), _f64(acc)
        self.lib.g2o_predict(_sz(len(pos)), pos.ctypes.data_as(C.c_void_p), vel.ctypes.data_as(C.c_void_p),
                             acc.ctypes.data_as(C.c_void_p), C.c_double(dt))
        return pos, vel

    def autotune(self, build_time, hist, min_i=1, max_i=128, cur=8):
        h = _f64(hist)
        return int(self.lib.g2o_autotune(C.c_double(build_time), _sz(len(h)), h.ctypes.data_as(C.c_void_p),
                                         _sz(min_i), _sz(max_i), _sz(cur)))


def force_error(acc, ref):
    """Nearest-rank relative-error statistics exactly as gravity.cpp:67-90."""
    acc, ref = np.asarray(acc, np.float64), np.asarray(ref, np.float64)
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
