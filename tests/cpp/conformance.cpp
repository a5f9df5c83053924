// C++ conformance suite for include/g2/gravitree.hpp (SURVEY §8b "Wrapper").
//
// The reference's own unit tests (proj/tests/test_tree.cpp, test_gravity.cpp, test_dynamics.cpp,
// test_perflab.cpp) restated against the B200 library through the reference's names: with
//     namespace gravitree = g2;
// the test bodies read as they do upstream.  Where the reference asserts FP64-exact equality of
// accelerations, the FP32 walk gets the documented tolerance variant; trees, events
// and error types are checked exactly.  Exit status 0 iff every check passes.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <functional>
#include <numeric>
#include <string>
#include <vector>

#include "g2/gravitree.hpp"

namespace gravitree = g2;
using gravitree::Vec3;

namespace {
int g_failed = 0, g_checks = 0;
#define CHECK(c)                                                                    \
    do {                                                                            \
        ++g_checks;                                                                 \
        if (!(c)) {                                                                 \
            ++g_failed;                                                             \
            std::fprintf(stderr, "  FAILED %s:%d: %s\n", __FILE__, __LINE__, #c);   \
        }                                                                           \
    } while (0)
template <class E, class F>
bool throws(F f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}
struct Case {
    const char* name;
    std::function<void()> body;
};
std::vector<Case>& cases() {
    static std::vector<Case> c;
    return c;
}
struct Reg {
    Reg(const char* n, std::function<void()> f) { cases().push_back({n, std::move(f)}); }
};
#define TEST_CASE(id, name) static void id(); static Reg reg_##id(name, id); static void id()

// uniform cube with masses in [0.5, 1.5] (test_support.hpp:14-23 shape; own counter-based RNG)
gravitree::ParticleSystem random_cloud(std::size_t n, std::uint64_t seed, double half = 1.0) {
    gravitree::ParticleSystem s(n);
    std::uint64_t x = seed * 0x9E3779B97F4A7C15ull + 1;
    auto u = [&] {
        x ^= x << 13, x ^= x >> 7, x ^= x << 17;
        return double(x >> 11) * 0x1.0p-53;
    };
    for (std::size_t i = 0; i < n; ++i) {
        s.mass[i] = 0.5 + u();
        s.pos[i] = {half * (2 * u() - 1), half * (2 * u() - 1), half * (2 * u() - 1)};
    }
    return s;
}
gravitree::ParticleSystem circular_binary() {  // test_support.hpp:51-60
    gravitree::ParticleSystem s(2);
    s.mass = {0.5, 0.5};
    const double v = 0.5;
    s.pos[0] = {-0.5, 0, 0}, s.pos[1] = {0.5, 0, 0};
    s.vel[0] = {0, -v, 0}, s.vel[1] = {0, v, 0};
    return s;
}
}  // namespace

// ---- test_tree.cpp -----------------------------------------------------------------------------
TEST_CASE(tree_single, "single particle -> one leaf cell (test_tree.cpp:73-84)") {
    gravitree::ParticleSystem s(1);
    s.mass[0] = 2.0, s.pos[0] = {0.3, -0.2, 0.1};
    gravitree::GravityEngine eng(gravitree::GravParams{});
    eng.build(s);
    const auto t = eng.tree();
    CHECK(t.cells.size() == 1);
    CHECK(t.cells[0].is_leaf() && t.cells[0].count == 1);
    CHECK(t.nodes[0].mass == 2.0);
}

TEST_CASE(tree_octants, "8 octants, leaf_cap 1 -> 9 cells, 8 leaves (test_tree.cpp:86-103)") {
    gravitree::ParticleSystem s(8);
    int i = 0;
    for (int a : {-1, 1})
        for (int b : {-1, 1})
            for (int c : {-1, 1}) s.mass[i] = 1.0, s.pos[i++] = {0.5 * a, 0.5 * b, 0.5 * c};
    gravitree::EngineConfig cfg;
    cfg.leaf_cap = 1;
    gravitree::GravityEngine eng(gravitree::GravParams{}, cfg);
    eng.build(s);
    const auto t = eng.tree();
    CHECK(t.cells.size() == 9);
    CHECK(t.root().child_count == 8);
    int leaves = 0;
    for (const auto& c : t.cells) leaves += c.is_leaf() ? 1 : 0;
    CHECK(leaves == 8);
}

TEST_CASE(tree_invariants, "random cloud: sorted keys, bijective perm, leaves cover n (test_tree.cpp:105-152)") {
    const auto s = random_cloud(1000, 7);
    gravitree::GravityEngine eng(gravitree::GravParams{});
    eng.build(s);
    const auto t = eng.tree();
    CHECK(std::is_sorted(t.keys.begin(), t.keys.end()));
    std::vector<int> seen(s.n(), 0);
    for (auto p : t.perm) ++seen.at(p);
    CHECK(std::all_of(seen.begin(), seen.end(), [](int v) { return v == 1; }));
    for (std::size_t k = 0; k < s.n(); ++k) CHECK(t.rank[t.perm[k]] == k);
    std::size_t covered = 0;
    for (const auto& c : t.cells) covered += c.is_leaf() ? c.count : 0;
    CHECK(covered == s.n());
    const double m = std::accumulate(s.mass.begin(), s.mass.end(), 0.0);
    Vec3 w;
    for (std::size_t k = 0; k < s.n(); ++k) w += s.mass[k] * s.pos[k];
    CHECK(std::abs(t.nodes[0].mass - m) <= 1e-12 * m);
    CHECK(((1.0 / m) * w - t.nodes[0].com).norm() < 1e-12);
    for (std::size_t c = 0; c < t.cells.size(); ++c)  // b_J >= every member distance (test_tree.cpp:154-164)
        for (std::uint32_t k = t.cells[c].first; k < t.cells[c].first + t.cells[c].count; ++k)
            CHECK((s.pos[t.perm[k]] - t.nodes[c].com).norm() <= t.nodes[c].extent * (1 + 1e-12));
}

TEST_CASE(tree_determinism, "rebuild determinism (test_gravity.cpp:231-240)") {
    const auto s = random_cloud(5000, 11);
    gravitree::GravityEngine a(gravitree::GravParams{}), b(gravitree::GravParams{});
    a.build(s), b.build(s);
    const auto ta = a.tree(), tb = b.tree();
    CHECK(ta.keys == tb.keys && ta.perm == tb.perm);
    bool same = ta.cells.size() == tb.cells.size();
    for (std::size_t c = 0; same && c < ta.cells.size(); ++c)
        same = ta.nodes[c].mass == tb.nodes[c].mass && ta.nodes[c].com.x == tb.nodes[c].com.x &&
               ta.nodes[c].extent == tb.nodes[c].extent && ta.cells[c].first == tb.cells[c].first;
    CHECK(same);
}

// ---- test_gravity.cpp --------------------------------------------------------------------------
TEST_CASE(direct_pairwise, "direct sum: two bodies, Newton III, zero-softening singularity (test_gravity.cpp:30-85)") {
    gravitree::ParticleSystem s(2);
    s.mass = {1.0, 1.0}, s.pos[0] = {0, 0, 0}, s.pos[1] = {1, 0, 0};
    const auto r = gravitree::direct_sum(s, gravitree::GravParams{});
    CHECK(r.acc[0].x == 1.0 && r.acc[1].x == -1.0);
    gravitree::GravParams soft;
    soft.eps = 1.0;
    const auto q = gravitree::direct_sum(s, soft);
    CHECK(std::abs(q.acc[0].x - std::pow(2.0, -1.5)) < 1e-15);
    CHECK(gravitree::count_walk_ops({2, 0, 0}).fp_fma == 18);
    s.pos[1] = s.pos[0];
    CHECK(throws<gravitree::singularity_error>([&] { gravitree::direct_sum(s, gravitree::GravParams{}); }));
}

TEST_CASE(walk_two_body, "two-body walk == direct sum (test_gravity.cpp:187-200; FP32 walk: 1e-6)") {
    gravitree::ParticleSystem s(2);
    s.mass = {1.0, 3.0}, s.pos[0] = {0.1, 0.2, 0.3}, s.pos[1] = {0.9, -0.4, 0.5};
    gravitree::GravityEngine eng(gravitree::GravParams{});
    eng.build(s);
    eng.bootstrap(s);
    eng.evaluate(s);
    const auto ref = gravitree::direct_sum(s, gravitree::GravParams{});
    for (int i = 0; i < 2; ++i) CHECK((s.acc[i] - ref.acc[i]).norm() <= 1e-6 * ref.acc[i].norm());
}

TEST_CASE(walk_accuracy, "p99 < 1e-3 at dacc 2^-20, median monotone over dacc (test_gravity.cpp:202-259)") {
    auto s = random_cloud(4000, 3);
    gravitree::GravParams p;
    p.eps = 0.01;
    const auto ref = gravitree::direct_sum(s, p);
    gravitree::GravityEngine eng(p);
    eng.build(s);
    eng.bootstrap(s);
    double prev = 1e300;
    std::uint64_t prev_inter = 0;
    for (int k : {3, 6, 9, 12, 15, 20}) {
        eng.params().dacc = std::ldexp(1.0, -k);
        const auto ev = eng.evaluate(s);
        const auto e = gravitree::force_error(s.acc, ref.acc);
        CHECK(e.median < prev);
        CHECK(ev.interactions > prev_inter);  // interactions rise as dacc tightens (test_gravity.cpp:300-321)
        prev = e.median, prev_inter = ev.interactions;
        if (k == 20) CHECK(e.p99 < 1e-3);
    }
}

TEST_CASE(walk_capacity, "results do not depend on list capacity (test_gravity.cpp:213-229; FP32: 1e-6)") {
    auto s = random_cloud(3000, 5);
    gravitree::GravParams p;
    p.eps = 0.01;
    std::vector<Vec3> first;
    gravitree::TraversalEvents ev0;
    for (std::size_t cap : {32u, 256u, 1024u}) {
        gravitree::EngineConfig cfg;
        cfg.list_capacity = cap;
        gravitree::GravityEngine eng(p, cfg);
        eng.build(s);
        eng.bootstrap(s);
        const auto ev = eng.evaluate(s);
        if (first.empty()) {
            first = s.acc, ev0 = ev;
            continue;
        }
        CHECK(ev == ev0);
        CHECK(gravitree::force_error(s.acc, first).max < 1e-6);
    }
}

TEST_CASE(walk_frontier_cap, "frontier cap 2 -> resource_error (test_gravity.cpp:261-272)") {
    auto s = random_cloud(2000, 9);
    gravitree::EngineConfig cfg;
    cfg.frontier_cap = 2;
    gravitree::GravityEngine eng(gravitree::GravParams{}, cfg);
    eng.build(s);
    CHECK(throws<gravitree::resource_error>([&] { eng.evaluate(s); }));
}

TEST_CASE(engine_contracts, "config and call-order errors, count_ops=false (engine.cpp:13-35, traversal.cpp:155)") {
    auto s = random_cloud(100, 1);
    CHECK(throws<gravitree::data_error>([] {
        gravitree::EngineConfig c;
        c.group_size = 0;
        gravitree::GravityEngine e(gravitree::GravParams{}, c);
    }));
    CHECK(throws<gravitree::data_error>([] {
        gravitree::GravParams p;
        p.dacc = 0.0;
        gravitree::GravityEngine e(p);
    }));
    gravitree::GravityEngine fresh(gravitree::GravParams{});
    CHECK(!fresh.has_tree());
    CHECK(throws<gravitree::data_error>([&] { fresh.evaluate(s); }));
    gravitree::EngineConfig quiet;
    quiet.count_ops = false;
    gravitree::GravityEngine eng(gravitree::GravParams{}, quiet);
    eng.build(s);
    CHECK(eng.has_tree());
    CHECK(eng.evaluate(s) == gravitree::TraversalEvents{});
    // engine.cpp:33-35: an empty target span walks nothing and leaves acc alone; a potential span
    // that does not cover the system is a data_error (before any walk)
    gravitree::GravityEngine counted(gravitree::GravParams{});
    counted.build(s);
    for (auto& a : s.acc) a = Vec3{7.0, 7.0, 7.0};
    const std::vector<std::uint32_t> none;
    CHECK(counted.evaluate(s, std::span<const std::uint32_t>(none)) == gravitree::TraversalEvents{});
    bool untouched = true;
    for (const auto& a : s.acc) untouched = untouched && a.x == 7.0 && a.y == 7.0 && a.z == 7.0;
    CHECK(untouched);
    std::vector<double> short_pot(10);
    const std::vector<std::uint32_t> some{1, 2, 3};
    CHECK(throws<gravitree::data_error>([&] { counted.evaluate(s, std::span<const std::uint32_t>(some), short_pot); }));
    CHECK(throws<gravitree::data_error>([&] { counted.evaluate(s, std::span<double>(short_pot)); }));
}

// ---- test_dynamics.cpp -------------------------------------------------------------------------
TEST_CASE(sim_circular_orbit, "circular orbit holds its radius over one period (test_dynamics.cpp:125-139)") {
    gravitree::GravParams p;
    p.dacc = 0x1.0p-20;
    gravitree::StepScheme sc;
    sc.adaptive = false;
    sc.dt_max = 6.283185307179586 / 1000.0;
    gravitree::Simulation sim(circular_binary(), p, sc);
    sim.init();
    bool ok = true;
    for (int k = 0; k < 1000; ++k) {
        sim.step();
        const auto& st = sim.system();
        ok = ok && std::abs((st.pos[1] - st.pos[0]).norm() - 1.0) < 0.01;
    }
    CHECK(ok);
}

TEST_CASE(sim_momentum, "symmetric static configuration conserves momentum (test_dynamics.cpp:176-196)") {
    gravitree::ParticleSystem s(8);
    int i = 0;
    for (int a : {-1, 1})
        for (int b : {-1, 1})
            for (int c : {-1, 1}) s.mass[i] = 1.0, s.pos[i++] = {0.5 * a, 0.5 * b, 0.5 * c};
    gravitree::GravParams p;
    p.eps = 0.1;
    gravitree::StepScheme sc;
    sc.dt_max = 0.01;
    gravitree::Simulation sim(s, p, sc);
    sim.init();
    const auto r = sim.step();
    Vec3 mom;
    const auto& st = sim.system();
    for (int k = 0; k < 8; ++k) mom += st.mass[k] * st.vel[k];
    CHECK(mom.norm() < 1e-12);
    CHECK(r.timings.total() <= r.wall_seconds * (1 + 1e-9) + 1e-9);  // test_dynamics.cpp:198-214
    CHECK(sim.initialized());
}

// ---- test_perflab.cpp --------------------------------------------------------------------------
TEST_CASE(op_counters, "costing constants, flops weights, speed-up fixed points (test_perflab.cpp:16-95)") {
    const auto c = gravitree::count_walk_ops({1, 1, 1});
    CHECK(c.fp_fma == 9 && c.fp_add == 5 && c.fp_mul == 5 && c.fp_rsqrt == 1 && c.integer == 16);
    gravitree::OpCounters f;
    f.fp_fma = 1;
    CHECK(gravitree::flops_estimate(f, 1.0) == 2.0);
    gravitree::OpCounters s;
    s.fp_add = 10;
    CHECK(std::abs(gravitree::predict_speedup(s, {}) - 1.5) < 1e-15);
    s.integer = 10;
    CHECK(std::abs(gravitree::predict_speedup(s, {}) - 3.0) < 1e-15);
    CHECK(throws<gravitree::data_error>([] { gravitree::predict_speedup({}, {}); }));
}

int main() {
    for (const auto& c : cases()) {
        const int before = g_failed;
        try {
            c.body();
        } catch (const std::exception& e) {
            ++g_failed;
            std::fprintf(stderr, "  FAILED %s: unexpected exception: %s\n", c.name, e.what());
        }
        std::printf("%s %s\n", g_failed == before ? "ok  " : "FAIL", c.name);
    }
    std::printf("%zu cases, %d checks, %d failed\n", cases().size(), g_checks, g_failed);
    return g_failed ? 1 : 0;
}
