// g2/gravitree.hpp -- header-only C++20 mirror of gravitree's operator API over the g2 C ABI.
//
// SURVEY §8b "Wrapper": the reference's types and classes under the same names (Vec3,
// ParticleSystem, GravParams, EngineConfig, StepScheme, TunerConfig, TraversalEvents, OpCounters,
// Octree, GravityEngine, Simulation, direct_sum, force_error, count_walk_ops, ...) with the same
// exception types, so code written against `gravitree::` compiles against the B200 library with
//     namespace gravitree = g2;
// Every numerical call goes to libg2.so (sm_100a); this header only marshals std::vector<Vec3>
// (three doubles, standard layout: the C ABI's double[3n]) and maps status codes to exceptions.
// Reference declarations: particle_system.hpp:14-57, octree.hpp:14-42, engine.hpp:14-66,
// integrator.hpp:14-91, op_counters.hpp:9-88, gravity.hpp:36-53, errors.hpp:8-23.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "g2/capi.h"

namespace g2 {

// ---- errors (errors.hpp:8-23) -------------------------------------------------------------
class data_error : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};
class resource_error : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};
class singularity_error : public data_error {
public:
    using data_error::data_error;
};

inline void check(int rc) {
    if (rc == G2_OK) return;
    const std::string m = g2_last_error();
    if (rc == G2_SINGULARITY) throw singularity_error(m);
    if (rc == G2_DATA_ERROR) throw data_error(m);
    if (rc == G2_RESOURCE_ERROR) throw resource_error(m);
    throw std::runtime_error(m);
}

// ---- value types ---------------------------------------------------------------------------
struct Vec3 {  // vec3.hpp: three doubles
    double x = 0.0, y = 0.0, z = 0.0;
    Vec3& operator+=(const Vec3& o) { return x += o.x, y += o.y, z += o.z, *this; }
    friend Vec3 operator+(Vec3 a, const Vec3& b) { return a += b; }
    friend Vec3 operator-(const Vec3& a, const Vec3& b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
    friend Vec3 operator*(double s, const Vec3& a) { return {s * a.x, s * a.y, s * a.z}; }
    double norm2() const { return x * x + y * y + z * z; }
    double norm() const { return std::sqrt(norm2()); }
};
static_assert(sizeof(Vec3) == 3 * sizeof(double), "Vec3 must be the C ABI's double[3]");

struct ParticleSystem {  // particle_system.hpp:14-49
    std::vector<double> mass;
    std::vector<Vec3> pos, vel, acc;
    std::vector<double> acc_old_mag;
    std::vector<std::uint8_t> level;
    double time = 0.0;
    ParticleSystem() = default;
    explicit ParticleSystem(std::size_t n) { resize(n); }
    std::size_t n() const { return mass.size(); }
    void resize(std::size_t n) {
        mass.assign(n, 0.0), pos.assign(n, Vec3{}), vel.assign(n, Vec3{}), acc.assign(n, Vec3{});
        acc_old_mag.assign(n, 0.0), level.assign(n, 0);
    }
};

struct GravParams {  // particle_system.hpp:53-57
    double G = 1.0, eps = 0.0, dacc = 0.001953125;
};
struct EngineConfig {  // engine.hpp:14-23
    std::size_t leaf_cap = 8, group_size = 32, list_capacity = 1024, frontier_cap = 0;
    bool count_ops = true;
    double bootstrap_theta = 0.5;
    std::size_t bootstrap_direct_limit = 65536;
    unsigned threads = 0;
};
struct StepScheme {  // integrator.hpp:18-23
    double eta = 0.5, dt_max = 0.0625;
    bool adaptive = true;
    int fixed_level = 0;
};
struct TunerConfig {  // rebuild_tuner.hpp:9-13
    std::size_t min_interval = 1, max_interval = 128, initial_interval = 8;
};
struct TraversalEvents {  // op_counters.hpp:33-46
    std::uint64_t interactions = 0, mac_evals = 0, list_pushes = 0;
    TraversalEvents& operator+=(const TraversalEvents& o) {
        return interactions += o.interactions, mac_evals += o.mac_evals, list_pushes += o.list_pushes, *this;
    }
    friend bool operator==(const TraversalEvents&, const TraversalEvents&) = default;
};
struct PhaseTimings {  // phase_timings.hpp:6-23 (device seconds)
    double walk_tree = 0.0, calc_node = 0.0, make_tree = 0.0, predict = 0.0, correct = 0.0;
    double total() const { return walk_tree + calc_node + make_tree + predict + correct; }
};
struct StepResult {  // integrator.hpp:43-50
    PhaseTimings timings;
    TraversalEvents events;
    std::size_t active = 0, rebuild_interval = 0;
    bool rebuilt = false;
    double wall_seconds = 0.0;
};
struct Cube {  // octree bounding cube
    Vec3 center;
    double half = 0.0;
};
struct Cell {  // octree.hpp:14-22
    std::uint32_t first_child = 0, child_count = 0, first = 0, count = 0;
    std::uint8_t depth = 0;
    bool is_leaf() const { return child_count == 0; }
};
struct NodeAttr {  // octree.hpp:26-30
    double mass = 0.0;
    Vec3 com;
    double extent = 0.0;
};
struct Octree {  // octree.hpp:32-42
    Cube bbox;
    std::vector<std::uint64_t> keys;
    std::vector<std::uint32_t> perm, rank;
    std::vector<Cell> cells;
    std::vector<NodeAttr> nodes;
    std::size_t leaf_cap = 8;
    const Cell& root() const { return cells.front(); }
};

// ---- op counters (op_counters.hpp:9-88, op_counters.cpp:7-28): host arithmetic ------------
struct OpCounters {
    std::uint64_t integer = 0, fp_fma = 0, fp_add = 0, fp_mul = 0, fp_rsqrt = 0;
    std::uint64_t fp_core() const { return fp_fma + fp_add + fp_mul; }
    std::uint64_t total() const { return integer + fp_core() + fp_rsqrt; }
};
inline constexpr OpCounters kInteractionCost{0, 9, 3, 2, 1};
inline constexpr OpCounters kMacEvalCost{12, 0, 2, 3, 0};
inline constexpr OpCounters kListPushCost{4, 0, 0, 0, 0};
inline OpCounters count_walk_ops(const TraversalEvents& e) {
    OpCounters c;
    c.integer = kInteractionCost.integer * e.interactions + kMacEvalCost.integer * e.mac_evals +
                kListPushCost.integer * e.list_pushes;
    c.fp_fma = kInteractionCost.fp_fma * e.interactions + kMacEvalCost.fp_fma * e.mac_evals;
    c.fp_add = kInteractionCost.fp_add * e.interactions + kMacEvalCost.fp_add * e.mac_evals;
    c.fp_mul = kInteractionCost.fp_mul * e.interactions + kMacEvalCost.fp_mul * e.mac_evals;
    c.fp_rsqrt = kInteractionCost.fp_rsqrt * e.interactions;
    return c;
}
inline double flops_estimate(const OpCounters& c, double seconds) {
    if (!(seconds > 0.0)) throw data_error("flops_estimate: elapsed time must be positive");
    return (2.0 * double(c.fp_fma) + double(c.fp_add) + double(c.fp_mul) + 4.0 * double(c.fp_rsqrt)) / seconds;
}
struct HardwareRatios {
    double peak_ratio = 1.5, bandwidth_ratio = 1.23;
};
inline double predict_speedup(const OpCounters& c, const HardwareRatios& hw) {
    const double f = double(c.fp_core()), i = double(c.integer);
    if (f == 0.0 && i == 0.0) throw data_error("predict_speedup: no counted instructions");
    return hw.peak_ratio * (i + f) / std::max(i, f);
}

namespace detail {
inline g2_grav_params c(const GravParams& p) { return {p.G, p.eps, p.dacc}; }
inline g2_engine_config c(const EngineConfig& e) {
    return {e.leaf_cap, e.group_size, e.list_capacity, e.frontier_cap, e.count_ops ? 1 : 0, e.bootstrap_theta,
            e.bootstrap_direct_limit, e.threads};
}
inline g2_step_scheme c(const StepScheme& s) { return {s.eta, s.dt_max, s.adaptive ? 1 : 0, s.fixed_level}; }
inline g2_tuner_config c(const TunerConfig& t) { return {t.min_interval, t.max_interval, t.initial_interval}; }
inline TraversalEvents ev(const g2_events& e) { return {e.interactions, e.mac_evals, e.list_pushes}; }
inline const double* d(const std::vector<Vec3>& v) { return v.empty() ? nullptr : &v[0].x; }
inline double* d(std::vector<Vec3>& v) { return v.empty() ? nullptr : &v[0].x; }
template <class Size, class Get>
Octree fetch_tree(Size size, Get get, std::size_t leaf_cap) {
    std::size_t n = 0, nc = 0;
    check(size(&n, &nc));
    Octree t;
    t.leaf_cap = leaf_cap;
    t.keys.resize(n), t.perm.resize(n), t.rank.resize(n), t.cells.resize(nc), t.nodes.resize(nc);
    std::vector<std::uint32_t> c4(4 * nc);
    std::vector<std::uint8_t> dep(nc);
    std::vector<double> n5(5 * nc), bb(4);
    check(get(bb.data(), t.keys.data(), t.perm.data(), t.rank.data(), c4.data(), dep.data(), n5.data()));
    t.bbox = Cube{{bb[0], bb[1], bb[2]}, bb[3]};
    for (std::size_t i = 0; i < nc; ++i) {
        t.cells[i] = Cell{c4[4 * i], c4[4 * i + 1], c4[4 * i + 2], c4[4 * i + 3], dep[i]};
        t.nodes[i] = NodeAttr{n5[5 * i], {n5[5 * i + 1], n5[5 * i + 2], n5[5 * i + 3]}, n5[5 * i + 4]};
    }
    return t;
}
}  // namespace detail

// ---- GravityEngine (engine.hpp:29-66) -------------------------------------------------------
class GravityEngine {
public:
    explicit GravityEngine(GravParams params, EngineConfig config = {}, int device = 0)
        : params_(params), pushed_(params), config_(config) {
        const g2_grav_params gp = detail::c(params);
        const g2_engine_config gc = detail::c(config);
        check(g2_engine_create(&gp, &gc, device, &h_));
    }
    ~GravityEngine() { g2_engine_destroy(h_); }
    GravityEngine(const GravityEngine&) = delete;
    GravityEngine& operator=(const GravityEngine&) = delete;

    void build(const ParticleSystem& s) { check(g2_engine_build(h_, s.n(), s.mass.data(), detail::d(s.pos))); }
    void build_structure(const ParticleSystem& s) {
        check(g2_engine_build_structure(h_, s.n(), s.mass.data(), detail::d(s.pos)));
    }
    void refresh(const ParticleSystem& s) { check(g2_engine_refresh(h_, s.n(), s.mass.data(), detail::d(s.pos))); }
    bool has_tree() const { return g2_engine_has_tree(h_) != 0; }
    // a host copy of the device tree (keys, perm, rank, cells, nodes: bit-identical to build_tree)
    Octree tree() const {
        return detail::fetch_tree([&](std::size_t* n, std::size_t* nc) { return g2_engine_tree_size(h_, n, nc); },
                                  [&](auto... a) { return g2_engine_get_tree(h_, a...); }, config_.leaf_cap);
    }
    const GravParams& params() const { return params_; }
    GravParams& params() { return params_; }  // mutable like the reference's; pushed before the next call
    const EngineConfig& config() const { return config_; }

    TraversalEvents evaluate(ParticleSystem& s, std::span<const std::uint32_t> targets, std::span<double> pot = {}) {
        // engine.cpp:32-35: an empty target span walks nothing (a null data() would mean "all
        // particles" at the C ABI), and pot must cover the system (the library writes pot[target])
        if (!has_tree()) throw data_error("GravityEngine::evaluate: no tree built");
        if (!pot.empty() && pot.size() != s.n())
            throw data_error("GravityEngine::evaluate: potential span must cover the system");
        if (targets.empty()) return {};
        sync_params();
        g2_events e{};
        check(g2_engine_evaluate(h_, s.n(), s.mass.data(), detail::d(s.pos), s.acc_old_mag.data(), targets.size(),
                                 targets.data(), detail::d(s.acc), pot.empty() ? nullptr : pot.data(), &e));
        return detail::ev(e);
    }
    TraversalEvents evaluate(ParticleSystem& s, std::span<double> pot = {}) {
        if (!has_tree()) throw data_error("GravityEngine::evaluate: no tree built");
        if (!pot.empty() && pot.size() != s.n())
            throw data_error("GravityEngine::evaluate: potential span must cover the system");
        sync_params();
        g2_events e{};
        check(g2_engine_evaluate(h_, s.n(), s.mass.data(), detail::d(s.pos), s.acc_old_mag.data(), 0, nullptr,
                                 detail::d(s.acc), pot.empty() ? nullptr : pot.data(), &e));
        return detail::ev(e);
    }
    TraversalEvents bootstrap(ParticleSystem& s) {
        sync_params();
        g2_events e{};
        check(g2_engine_bootstrap(h_, s.n(), s.mass.data(), detail::d(s.pos), detail::d(s.acc),
                                  s.acc_old_mag.data(), &e));
        return detail::ev(e);
    }

private:
    void sync_params() {
        if (params_.G == pushed_.G && params_.eps == pushed_.eps && params_.dacc == pushed_.dacc) return;
        const g2_grav_params gp = detail::c(params_);
        check(g2_engine_set_params(h_, &gp));
        pushed_ = params_;
    }
    g2_engine* h_ = nullptr;
    GravParams params_, pushed_;
    EngineConfig config_;
};

// ---- Simulation (integrator.hpp:54-91): device-resident state, system() copies it out --------
class Simulation {
public:
    Simulation(ParticleSystem system, GravParams params, StepScheme scheme, EngineConfig engine_config = {},
               TunerConfig tuner_config = {}, int device = 0)
        : system_(std::move(system)), params_(params), scheme_(scheme), config_(engine_config) {
        const g2_grav_params gp = detail::c(params);
        const g2_step_scheme gs = detail::c(scheme);
        const g2_engine_config gc = detail::c(engine_config);
        const g2_tuner_config gt = detail::c(tuner_config);
        check(g2_sim_create(system_.n(), system_.mass.data(), detail::d(system_.pos), detail::d(system_.vel), &gp,
                            &gs, &gc, &gt, device, &h_));
    }
    ~Simulation() { g2_sim_destroy(h_); }
    Simulation(const Simulation&) = delete;
    Simulation& operator=(const Simulation&) = delete;

    void init() {
        check(g2_sim_init(h_));
        initialized_ = true;
        stale_ = true;
    }
    StepResult step() {
        g2_step_result r{};
        check(g2_sim_step(h_, &r));
        stale_ = true;
        return {{r.walk_tree, r.calc_node, r.make_tree, r.predict, r.correct},
                detail::ev(r.events),
                r.active,
                r.rebuild_interval,
                r.rebuilt != 0,
                r.wall_seconds};
    }
    // the state in original particle order (copied from the device on first access after a step)
    const ParticleSystem& system() {
        if (stale_) {
            check(g2_sim_get_state(h_, detail::d(system_.pos), detail::d(system_.vel), detail::d(system_.acc),
                                   system_.acc_old_mag.data(), system_.level.data(), &system_.time));
            stale_ = false;
        }
        return system_;
    }
    Octree tree() const {  // engine().tree() of the last rebuild
        return detail::fetch_tree([&](std::size_t* n, std::size_t* nc) { return g2_sim_tree_size(h_, n, nc); },
                                  [&](auto... a) { return g2_sim_get_tree(h_, a...); }, config_.leaf_cap);
    }
    const StepScheme& scheme() const { return scheme_; }
    double time() { return system().time; }
    bool initialized() const { return initialized_; }
    void set_fixed_rebuild_interval(std::size_t k) { check(g2_sim_set_fixed_rebuild_interval(h_, k)); }

private:
    g2_sim* h_ = nullptr;
    ParticleSystem system_;
    GravParams params_;
    StepScheme scheme_;
    EngineConfig config_;
    bool initialized_ = false, stale_ = false;
};

// ---- free functions (gravity.hpp:36-53) -----------------------------------------------------
struct DirectSumResult {
    std::vector<Vec3> acc;
    OpCounters ops;
};
// FP64 direct summation on the device, the reference's summation order (gravity.cpp:18-43)
inline DirectSumResult direct_sum(const ParticleSystem& s, const GravParams& p, unsigned /*threads*/ = 0,
                                  int device = 0) {
    DirectSumResult r;
    r.acc.resize(s.n());
    check(g2_direct_sum(s.n(), s.mass.data(), detail::d(s.pos), p.G, p.eps, device, detail::d(r.acc)));
    TraversalEvents ev;  // the reference's costing: n (n - 1) interactions (gravity.cpp:40-42)
    ev.interactions = std::uint64_t(s.n()) * (s.n() ? s.n() - 1 : 0);
    r.ops = count_walk_ops(ev);
    return r;
}
struct ForceErrorStats {
    double median = 0.0, p99 = 0.0, max = 0.0;
    std::size_t excluded = 0;
};
// nearest-rank relative-error statistics, zero references excluded (gravity.cpp:67-90)
inline ForceErrorStats force_error(const std::vector<Vec3>& tree_acc, const std::vector<Vec3>& oracle_acc) {
    if (tree_acc.size() != oracle_acc.size()) throw data_error("force_error: length mismatch");
    ForceErrorStats st;
    std::vector<double> err;
    err.reserve(tree_acc.size());
    for (std::size_t i = 0; i < tree_acc.size(); ++i) {
        const double rn = oracle_acc[i].norm();
        if (rn == 0.0) {
            ++st.excluded;
            continue;
        }
        err.push_back((tree_acc[i] - oracle_acc[i]).norm() / rn);
    }
    if (err.empty()) return st;
    std::sort(err.begin(), err.end());
    auto rank = [&](double pct) {
        const std::size_t k = std::size_t(std::ceil(pct / 100.0 * double(err.size())));
        return err[k ? k - 1 : 0];
    };
    st.median = rank(50.0), st.p99 = rank(99.0), st.max = err.back();
    return st;
}

}  // namespace g2
