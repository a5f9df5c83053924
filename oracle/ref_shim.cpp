// ORACLE / TEST INFRASTRUCTURE ONLY.
//
// extern "C" shim over the UNMODIFIED gravitree reference library, which
// oracle/Makefile compiles in place from /root/reference/proj/core/src into
// oracle/_ref/libgravitree_ref.so.  Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs may load it.  Nothing here
// is on the product path.
//
// Every entry point forwards to a public reference API:
//   sample_model            models.cpp:442-460
//   build_tree / calc_node  octree.cpp:51-106, 145-162
//   GravityEngine           engine.hpp:29-66, engine.cpp:13-103
//   direct_sum / force_error gravity.cpp:18-43, 67-90
//   make_group              traversal.cpp:16-38
//   predict/correct/block_level, Simulation   integrator.cpp:21-164
//   autotune_rebuild        rebuild_tuner.cpp:28-61
// Status codes: 0 ok, 3 data_error, 4 resource_error, 5 singularity_error.

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "gravitree/diagnostics.hpp"
#include "gravitree/engine.hpp"
#include "gravitree/snapshot.hpp"
#include "gravitree/errors.hpp"
#include "gravitree/gravity.hpp"
#include "gravitree/integrator.hpp"
#include "gravitree/models.hpp"
#include "gravitree/octree.hpp"
#include "gravitree/parallel.hpp"
#include "gravitree/rebuild_tuner.hpp"
#include "gravitree/traversal.hpp"

using namespace gravitree;

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const singularity_error& e) {
        g_err = e.what();
        return 5;
    } catch (const resource_error& e) {
        g_err = e.what();
        return 4;
    } catch (const data_error& e) {
        g_err = e.what();
        return 3;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

void load_system(ParticleSystem& s, std::size_t n, const double* mass, const double* pos, const double* vel,
                 const double* acc, const double* acc_old_mag) {
    s.resize(n);
    for (std::size_t i = 0; i < n; ++i) {
        s.mass[i] = mass[i];
        s.pos[i] = {pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]};
        if (vel) s.vel[i] = {vel[3 * i], vel[3 * i + 1], vel[3 * i + 2]};
        if (acc) s.acc[i] = {acc[3 * i], acc[3 * i + 1], acc[3 * i + 2]};
        if (acc_old_mag) s.acc_old_mag[i] = acc_old_mag[i];
    }
}

void store_vec(const std::vector<Vec3>& v, double* out) {
    for (std::size_t i = 0; i < v.size(); ++i) {
        out[3 * i] = v[i].x;
        out[3 * i + 1] = v[i].y;
        out[3 * i + 2] = v[i].z;
    }
}

struct TreeOut {
    Octree tree;
};

void copy_tree(const Octree& t, double* bbox4, std::uint64_t* keys, std::uint32_t* perm, std::uint32_t* rank,
               std::uint32_t* cells4, std::uint8_t* depth, double* nodes5) {
    if (bbox4) {
        bbox4[0] = t.bbox.center.x;
        bbox4[1] = t.bbox.center.y;
        bbox4[2] = t.bbox.center.z;
        bbox4[3] = t.bbox.half;
    }
    const std::size_t n = t.keys.size();
    if (keys) std::memcpy(keys, t.keys.data(), n * 8);
    if (perm) std::memcpy(perm, t.perm.data(), n * 4);
    if (rank) std::memcpy(rank, t.rank.data(), n * 4);
    for (std::size_t c = 0; c < t.cells.size(); ++c) {
        if (cells4) {
            cells4[4 * c] = t.cells[c].first_child;
            cells4[4 * c + 1] = t.cells[c].child_count;
            cells4[4 * c + 2] = t.cells[c].first;
            cells4[4 * c + 3] = t.cells[c].count;
        }
        if (depth) depth[c] = t.cells[c].depth;
        if (nodes5 && c < t.nodes.size()) {
            nodes5[5 * c] = t.nodes[c].mass;
            nodes5[5 * c + 1] = t.nodes[c].com.x;
            nodes5[5 * c + 2] = t.nodes[c].com.y;
            nodes5[5 * c + 3] = t.nodes[c].com.z;
            nodes5[5 * c + 4] = t.nodes[c].extent;
        }
    }
}

struct EngineHandle {
    GravityEngine engine;
    ParticleSystem system;
    EngineHandle(GravParams p, EngineConfig c) : engine(p, c) {}
};

struct SimHandle {
    std::unique_ptr<Simulation> sim;
};

}  // namespace

extern "C" {

const char* gtref_last_error() { return g_err.c_str(); }

unsigned gtref_resolve_threads(unsigned t) { return resolve_threads(t); }

int gtref_sample_model(const char* name, std::size_t n, std::uint64_t seed, double* mass, double* pos,
                       double* vel) {
    return guarded([&] {
        const ParticleSystem s = sample_model(name, n, seed);
        for (std::size_t i = 0; i < n; ++i) mass[i] = s.mass[i];
        store_vec(s.pos, pos);
        store_vec(s.vel, vel);
    });
}

// ---- trees -----------------------------------------------------------------
int gtref_tree_build(std::size_t n, const double* mass, const double* pos, std::size_t leaf_cap, int with_nodes,
                     void** out) {
    return guarded([&] {
        ParticleSystem s;
        load_system(s, n, mass, pos, nullptr, nullptr, nullptr);
        auto* h = new TreeOut{build_tree(s, leaf_cap, with_nodes != 0)};
        *out = h;
    });
}

int gtref_tree_calc_node(void* h, std::size_t n, const double* mass, const double* pos, unsigned threads) {
    return guarded([&] {
        ParticleSystem s;
        load_system(s, n, mass, pos, nullptr, nullptr, nullptr);
        calc_node(static_cast<TreeOut*>(h)->tree, s, threads);
    });
}

std::size_t gtref_tree_ncells(void* h) { return static_cast<TreeOut*>(h)->tree.cells.size(); }

void gtref_tree_get(void* h, double* bbox4, std::uint64_t* keys, std::uint32_t* perm, std::uint32_t* rank,
                    std::uint32_t* cells4, std::uint8_t* depth, double* nodes5) {
    copy_tree(static_cast<TreeOut*>(h)->tree, bbox4, keys, perm, rank, cells4, depth, nodes5);
}

void gtref_tree_free(void* h) { delete static_cast<TreeOut*>(h); }

int gtref_bounding_cube(std::size_t n, const double* pos, double* bbox4) {
    return guarded([&] {
        std::vector<Vec3> p(n);
        for (std::size_t i = 0; i < n; ++i) p[i] = {pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]};
        const Cube c = bounding_cube(p);
        bbox4[0] = c.center.x;
        bbox4[1] = c.center.y;
        bbox4[2] = c.center.z;
        bbox4[3] = c.half;
    });
}

// ---- gravity engine ----------------------------------------------------------
int gtref_engine_create(double G, double eps, double dacc, std::size_t leaf_cap, std::size_t group_size,
                        std::size_t list_capacity, std::size_t frontier_cap, int count_ops, double theta,
                        std::size_t direct_limit, unsigned threads, void** out) {
    return guarded([&] {
        GravParams p{G, eps, dacc};
        EngineConfig c;
        c.leaf_cap = leaf_cap;
        c.group_size = group_size;
        c.list_capacity = list_capacity;
        c.frontier_cap = frontier_cap;
        c.count_ops = count_ops != 0;
        c.bootstrap_theta = theta;
        c.bootstrap_direct_limit = direct_limit;
        c.threads = threads;
        *out = new EngineHandle(p, c);
    });
}

void gtref_engine_destroy(void* h) { delete static_cast<EngineHandle*>(h); }

int gtref_engine_build(void* h, std::size_t n, const double* mass, const double* pos, int with_nodes) {
    return guarded([&] {
        auto* e = static_cast<EngineHandle*>(h);
        load_system(e->system, n, mass, pos, nullptr, nullptr, nullptr);
        if (with_nodes)
            e->engine.build(e->system);
        else
            e->engine.build_structure(e->system);
    });
}

int gtref_engine_refresh(void* h, std::size_t n, const double* mass, const double* pos) {
    return guarded([&] {
        auto* e = static_cast<EngineHandle*>(h);
        load_system(e->system, n, mass, pos, nullptr, nullptr, nullptr);
        e->engine.refresh(e->system);
    });
}

std::size_t gtref_engine_ncells(void* h) { return static_cast<EngineHandle*>(h)->engine.tree().cells.size(); }

void gtref_engine_get_tree(void* h, double* bbox4, std::uint64_t* keys, std::uint32_t* perm, std::uint32_t* rank,
                           std::uint32_t* cells4, std::uint8_t* depth, double* nodes5) {
    copy_tree(static_cast<EngineHandle*>(h)->engine.tree(), bbox4, keys, perm, rank, cells4, depth, nodes5);
}

// targets == nullptr: all particles (GravityEngine::evaluate(system, pot)).
int gtref_engine_evaluate(void* h, std::size_t n, const double* mass, const double* pos,
                          const double* acc_old_mag, std::size_t n_targets, const std::uint32_t* targets,
                          double* acc_out, double* pot_out, std::uint64_t* events3) {
    return guarded([&] {
        auto* e = static_cast<EngineHandle*>(h);
        load_system(e->system, n, mass, pos, nullptr, acc_out, acc_old_mag);
        std::vector<double> pot(pot_out ? n : 0, 0.0);
        TraversalEvents ev;
        if (targets)
            ev = e->engine.evaluate(e->system, std::span<const std::uint32_t>(targets, n_targets), pot);
        else
            ev = e->engine.evaluate(e->system, pot);
        store_vec(e->system.acc, acc_out);
        if (pot_out)
            for (std::size_t i = 0; i < n; ++i) pot_out[i] = pot[i];
        if (events3) {
            events3[0] = ev.interactions;
            events3[1] = ev.mac_evals;
            events3[2] = ev.list_pushes;
        }
    });
}

int gtref_engine_bootstrap(void* h, std::size_t n, const double* mass, const double* pos, double* acc_out,
                           double* acc_old_mag_out, std::uint64_t* events3) {
    return guarded([&] {
        auto* e = static_cast<EngineHandle*>(h);
        load_system(e->system, n, mass, pos, nullptr, nullptr, nullptr);
        const TraversalEvents ev = e->engine.bootstrap(e->system);
        store_vec(e->system.acc, acc_out);
        for (std::size_t i = 0; i < n; ++i) acc_old_mag_out[i] = e->system.acc_old_mag[i];
        if (events3) {
            events3[0] = ev.interactions;
            events3[1] = ev.mac_evals;
            events3[2] = ev.list_pushes;
        }
    });
}

// Group spheres exactly as evaluate() forms them (engine.cpp:38-44 + make_group).
int gtref_groups(std::size_t n, const double* pos, const double* acc_old_mag, const std::uint32_t* rank,
                 std::size_t n_targets, const std::uint32_t* targets, std::size_t group_size, double* out5) {
    return guarded([&] {
        ParticleSystem s;
        s.resize(n);
        for (std::size_t i = 0; i < n; ++i) {
            s.pos[i] = {pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]};
            s.acc_old_mag[i] = acc_old_mag[i];
            s.mass[i] = 1.0;
        }
        std::vector<std::uint32_t> ordered(targets, targets + n_targets);
        std::sort(ordered.begin(), ordered.end(), [&](std::uint32_t a, std::uint32_t b) { return rank[a] < rank[b]; });
        const std::size_t ng = (ordered.size() + group_size - 1) / group_size;
        for (std::size_t g = 0; g < ng; ++g) {
            const std::size_t lo = g * group_size;
            const std::size_t cnt = std::min(group_size, ordered.size() - lo);
            const TraversalGroup grp = make_group(s, {ordered.data() + lo, cnt});
            out5[5 * g] = grp.center.x;
            out5[5 * g + 1] = grp.center.y;
            out5[5 * g + 2] = grp.center.z;
            out5[5 * g + 3] = grp.radius;
            out5[5 * g + 4] = grp.a_min;
        }
    });
}

int gtref_direct_sum(std::size_t n, const double* mass, const double* pos, double G, double eps, unsigned threads,
                     double* acc_out) {
    return guarded([&] {
        ParticleSystem s;
        load_system(s, n, mass, pos, nullptr, nullptr, nullptr);
        const DirectSumResult r = direct_sum(s, GravParams{G, eps, 0.001953125}, threads);
        store_vec(r.acc, acc_out);
    });
}

// write_snapshot / read_snapshot (snapshot.cpp:65-121) on flat arrays
int gtref_write_snapshot(const char* path, std::size_t n, const double* mass, const double* pos, const double* vel,
                         double time, double G, double eps) {
    return guarded([&] {
        ParticleSystem sys(n);
        sys.mass.assign(mass, mass + n);
        for (std::size_t i = 0; i < n; ++i) {
            sys.pos[i] = {pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]};
            sys.vel[i] = {vel[3 * i], vel[3 * i + 1], vel[3 * i + 2]};
        }
        sys.time = time;
        GravParams p;
        p.G = G, p.eps = eps;
        write_snapshot(path, sys, p);
    });
}
int gtref_read_snapshot(const char* path, std::size_t cap, double* mass, double* pos, double* vel, double* hdr4) {
    return guarded([&] {
        const Snapshot s = read_snapshot(path);
        const std::size_t n = s.system.n();
        hdr4[0] = double(n), hdr4[1] = s.system.time, hdr4[2] = s.G, hdr4[3] = s.eps;
        if (n > cap) return;
        for (std::size_t i = 0; i < n; ++i) {
            mass[i] = s.system.mass[i];
            pos[3 * i] = s.system.pos[i].x, pos[3 * i + 1] = s.system.pos[i].y, pos[3 * i + 2] = s.system.pos[i].z;
            vel[3 * i] = s.system.vel[i].x, vel[3 * i + 1] = s.system.vel[i].y, vel[3 * i + 2] = s.system.vel[i].z;
        }
    });
}

// compute_diagnostics (diagnostics.cpp:10-38) on a ParticleSystem built from flat arrays
int gtref_diagnostics(std::size_t n, const double* mass, const double* pos, const double* vel,
                      const double* acc_old_mag, double G, double eps, double dacc, unsigned threads, double* out7) {
    return guarded([&] {
        ParticleSystem sys;
        sys.mass.assign(mass, mass + n);
        sys.pos.resize(n), sys.vel.resize(n), sys.acc.assign(n, Vec3{});
        for (std::size_t i = 0; i < n; ++i) {
            sys.pos[i] = {pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]};
            sys.vel[i] = {vel[3 * i], vel[3 * i + 1], vel[3 * i + 2]};
        }
        sys.acc_old_mag.assign(n, 0.0);
        if (acc_old_mag) sys.acc_old_mag.assign(acc_old_mag, acc_old_mag + n);
        sys.level.assign(n, 0);
        GravParams p;
        p.G = G, p.eps = eps, p.dacc = dacc;
        const Diagnostics d = compute_diagnostics(sys, p, threads);
        out7[0] = d.kinetic, out7[1] = d.potential, out7[2] = d.total;
        out7[3] = d.momentum.x, out7[4] = d.momentum.y, out7[5] = d.momentum.z, out7[6] = d.virial_ratio;
    });
}

int gtref_force_error(std::size_t n, const double* acc, const double* ref, double* out4) {
    return guarded([&] {
        std::vector<Vec3> a(n), b(n);
        for (std::size_t i = 0; i < n; ++i) {
            a[i] = {acc[3 * i], acc[3 * i + 1], acc[3 * i + 2]};
            b[i] = {ref[3 * i], ref[3 * i + 1], ref[3 * i + 2]};
        }
        const ForceErrorStats s = force_error(a, b);
        out4[0] = s.median;
        out4[1] = s.p99;
        out4[2] = s.max;
        out4[3] = static_cast<double>(s.excluded);
    });
}

// ---- integrator free functions ------------------------------------------------
int gtref_block_level(double acc_mag, double eta, double dt_max, int adaptive, int fixed_level, double eps) {
    StepScheme s;
    s.eta = eta;
    s.dt_max = dt_max;
    s.adaptive = adaptive != 0;
    s.fixed_level = fixed_level;
    return block_level(acc_mag, s, eps);
}

int gtref_predict(std::size_t n, double* pos, double* vel, const double* acc, double dt) {
    return guarded([&] {
        ParticleSystem s;
        std::vector<double> m(n, 1.0);
        load_system(s, n, m.data(), pos, vel, acc, nullptr);
        predict(s, dt);
        store_vec(s.pos, pos);
        store_vec(s.vel, vel);
    });
}

int gtref_correct(std::size_t n, double* vel, double* acc, double* acc_old_mag, const double* new_acc, double dt) {
    return guarded([&] {
        ParticleSystem s;
        std::vector<double> m(n, 1.0), p(3 * n, 0.0);
        load_system(s, n, m.data(), p.data(), vel, acc, acc_old_mag);
        std::vector<Vec3> na(n);
        for (std::size_t i = 0; i < n; ++i) na[i] = {new_acc[3 * i], new_acc[3 * i + 1], new_acc[3 * i + 2]};
        correct(s, na, dt);
        store_vec(s.vel, vel);
        store_vec(s.acc, acc);
        for (std::size_t i = 0; i < n; ++i) acc_old_mag[i] = s.acc_old_mag[i];
    });
}

std::size_t gtref_autotune(double build_time, std::size_t n_hist, const double* hist, std::size_t min_i,
                           std::size_t max_i, std::size_t initial) {
    RebuildTuner t(TunerConfig{min_i, max_i, initial});
    t.record_build(build_time);
    for (std::size_t k = 0; k < n_hist; ++k) t.record_walk(hist[k]);
    return autotune_rebuild(t);
}

// ---- simulation ------------------------------------------------------------------
int gtref_sim_create(std::size_t n, const double* mass, const double* pos, const double* vel, double G, double eps,
                     double dacc, double eta, double dt_max, int adaptive, int fixed_level, std::size_t leaf_cap,
                     std::size_t group_size, unsigned threads, void** out) {
    return guarded([&] {
        ParticleSystem s;
        load_system(s, n, mass, pos, vel, nullptr, nullptr);
        StepScheme sc;
        sc.eta = eta;
        sc.dt_max = dt_max;
        sc.adaptive = adaptive != 0;
        sc.fixed_level = fixed_level;
        EngineConfig ec;
        ec.leaf_cap = leaf_cap;
        ec.group_size = group_size;
        ec.threads = threads;
        auto* h = new SimHandle;
        h->sim = std::make_unique<Simulation>(std::move(s), GravParams{G, eps, dacc}, sc, ec);
        *out = h;
    });
}

void gtref_sim_destroy(void* h) { delete static_cast<SimHandle*>(h); }

int gtref_sim_init(void* h) {
    return guarded([&] { static_cast<SimHandle*>(h)->sim->init(); });
}

int gtref_sim_set_fixed_rebuild_interval(void* h, std::size_t interval) {
    return guarded([&] { static_cast<SimHandle*>(h)->sim->set_fixed_rebuild_interval(interval); });
}

// out8: walk, calc, make, predict, correct, wall, active, rebuild_interval; flags: rebuilt; events3
int gtref_sim_step(void* h, double* out8, int* rebuilt, std::uint64_t* events3) {
    return guarded([&] {
        const StepResult r = static_cast<SimHandle*>(h)->sim->step();
        out8[0] = r.timings.walk_tree;
        out8[1] = r.timings.calc_node;
        out8[2] = r.timings.make_tree;
        out8[3] = r.timings.predict;
        out8[4] = r.timings.correct;
        out8[5] = r.wall_seconds;
        out8[6] = static_cast<double>(r.active);
        out8[7] = static_cast<double>(r.rebuild_interval);
        *rebuilt = r.rebuilt ? 1 : 0;
        events3[0] = r.events.interactions;
        events3[1] = r.events.mac_evals;
        events3[2] = r.events.list_pushes;
    });
}

// ---- all-active stepping loop (bench.py --impl reference / cpu_baseline) ----------------
// Simulation::step (integrator.cpp:97-164) with every particle at level 0 (StepScheme
// adaptive=false, fixed_level=0: all particles active every step, dt_block = dt_max) and the
// rebuild decision forced to "rebuild" -- the reference's own Simulation cannot rebuild every step
// (rebuild_tuner.hpp:26 requires >= 2 steps), and bench.py's workload rebuilds every step.  Every
// phase is the reference's public API on a resident ParticleSystem: predict (integrator.cpp:40-45),
// GravityEngine::build_structure + refresh (engine.cpp), evaluate on all active particles
// (engine.cpp:31-81) and the corrector loop of integrator.cpp:148-156.  Setup runs the reference's
// bootstrap (engine.cpp:89-103), as Simulation::init does.
struct LoopHandle {
    ParticleSystem system;
    GravityEngine engine;
    std::vector<std::uint32_t> active;
    LoopHandle(GravParams p, EngineConfig c) : engine(p, c) {}
};

int gtref_loop_create(std::size_t n, const double* mass, const double* pos, const double* vel, const double* acc,
                      const double* acc_old_mag, double G, double eps, double dacc, unsigned threads, void** out) {
    return guarded([&] {
        EngineConfig c;
        c.threads = threads;
        auto h = std::make_unique<LoopHandle>(GravParams{G, eps, dacc}, c);
        load_system(h->system, n, mass, pos, vel, acc, acc_old_mag);
        h->system.validate();
        if (!acc) h->engine.bootstrap(h->system);  // Simulation::init (integrator.cpp:69-79)
        h->active.resize(n);
        for (std::size_t i = 0; i < n; ++i) h->active[i] = static_cast<std::uint32_t>(i);
        *out = h.release();
    });
}

void gtref_loop_destroy(void* h) { delete static_cast<LoopHandle*>(h); }

// out6: predict, make_tree, calc_node, walk_tree, correct, total seconds; events3
int gtref_loop_step(void* hv, double dt, double* out6, std::uint64_t* events3) {
    return guarded([&] {
        using Clock = std::chrono::steady_clock;
        auto secs = [](Clock::time_point a) { return std::chrono::duration<double>(Clock::now() - a).count(); };
        auto* h = static_cast<LoopHandle*>(hv);
        ParticleSystem& s = h->system;
        const auto start = Clock::now();
        auto t0 = Clock::now();
        predict(s, dt);
        out6[0] = secs(t0);
        t0 = Clock::now();
        h->engine.build_structure(s);
        out6[1] = secs(t0);
        t0 = Clock::now();
        h->engine.refresh(s);
        out6[2] = secs(t0);
        std::vector<Vec3> acc_old(s.acc);  // every particle is active
        t0 = Clock::now();
        const TraversalEvents ev = h->engine.evaluate(s, h->active);
        out6[3] = secs(t0);
        t0 = Clock::now();
        for (std::size_t i = 0; i < s.n(); ++i) {
            s.vel[i] += (0.5 * dt) * (s.acc[i] - acc_old[i]);
            s.acc_old_mag[i] = s.acc[i].norm();
        }
        s.time += dt;
        out6[4] = secs(t0);
        out6[5] = secs(start);
        if (events3) {
            events3[0] = ev.interactions;
            events3[1] = ev.mac_evals;
            events3[2] = ev.list_pushes;
        }
    });
}

void gtref_loop_get_state(void* hv, double* pos, double* vel, double* acc, double* acc_old_mag) {
    const ParticleSystem& s = static_cast<LoopHandle*>(hv)->system;
    if (pos) store_vec(s.pos, pos);
    if (vel) store_vec(s.vel, vel);
    if (acc) store_vec(s.acc, acc);
    if (acc_old_mag)
        for (std::size_t i = 0; i < s.n(); ++i) acc_old_mag[i] = s.acc_old_mag[i];
}

void gtref_sim_get_state(void* h, double* pos, double* vel, double* acc, double* acc_old_mag, std::uint8_t* level,
                         double* time) {
    const ParticleSystem& s = static_cast<SimHandle*>(h)->sim->system();
    if (pos) store_vec(s.pos, pos);
    if (vel) store_vec(s.vel, vel);
    if (acc) store_vec(s.acc, acc);
    if (acc_old_mag)
        for (std::size_t i = 0; i < s.n(); ++i) acc_old_mag[i] = s.acc_old_mag[i];
    if (level)
        for (std::size_t i = 0; i < s.n(); ++i) level[i] = s.level[i];
    if (time) *time = s.time;
}

}  // extern "C"
